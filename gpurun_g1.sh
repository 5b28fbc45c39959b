mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/g1_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/g1_smoke.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "walk or hash or corridor or random" > gpurun_out/g1_parity.txt 2>&1; echo "rc=$?" >> gpurun_out/g1_parity.txt
timeout 600 python bench.py --steps 2 --warmup 1 --batches 200 --no-cpu > gpurun_out/g1_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/g1_bench.txt
timeout 300 python bench.py --workload c1 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/g1_bench_c1.txt 2>&1
timeout 300 python bench.py --workload c1 --exec cas --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/g1_bench_c1cas.txt 2>&1
tail -5 gpurun_out/g1_smoke.txt gpurun_out/g1_parity.txt gpurun_out/g1_bench.txt gpurun_out/g1_bench_c1.txt gpurun_out/g1_bench_c1cas.txt

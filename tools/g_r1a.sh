mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/a_pytest.txt
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/a_c1.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/a_c2.txt 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --exec cas --no-cpu --no-e2e > gpurun_out/a_c2cas.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.txt 2>&1

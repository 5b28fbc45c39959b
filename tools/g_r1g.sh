mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/g_pytest.txt
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g_c1.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/g_c2.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --exec cas > gpurun_out/g_c2cas.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk" -s 10 -c 1 -o gpurun_out/g_prog_c2 python tools/prog_run.py --workload c2 --batches 300 > gpurun_out/g_ncu.txt 2>&1

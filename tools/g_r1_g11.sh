mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not ndt" > gpurun_out/g11_parity.txt 2>&1; echo "rc=$?" >> gpurun_out/g11_parity.txt
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g11_c1.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/g11_c2.txt 2>&1

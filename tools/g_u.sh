mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/u_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/u_pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/u_c2.txt 2>&1

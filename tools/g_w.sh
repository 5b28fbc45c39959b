mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/w_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/w_pytest.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/w_c2.txt 2>&1
timeout 900 python bench.py --workload c3 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/w_c3.txt 2>&1

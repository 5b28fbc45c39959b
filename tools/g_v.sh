mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/v_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/v_pytest.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/v_c2.txt 2>&1

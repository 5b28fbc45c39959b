mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x -m gpu > gpurun_out/o_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/o_pytest.txt

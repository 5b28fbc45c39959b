mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider > gpurun_out/ah_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/ah_pytest.txt

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_exports.py -p no:cacheprovider > gpurun_out/r_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/r_pytest_all.txt

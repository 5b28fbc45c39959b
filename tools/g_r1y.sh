mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/y_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/y_pytest_all.txt

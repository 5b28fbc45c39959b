mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2a_smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2a_pytest.txt
timeout 600 python bench.py > gpurun_out/r2a_bench.txt 2>&1

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2g_all.txt 2>&1; echo "rc=$?" >> gpurun_out/r2g_all.txt
timeout 900 python bench.py > gpurun_out/r2g_bench.txt 2>&1

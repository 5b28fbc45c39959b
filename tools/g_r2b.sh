mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ndt.py -q -x -p no:cacheprovider > gpurun_out/r2b_ndt.txt 2>&1; echo "rc=$?" >> gpurun_out/r2b_ndt.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b_all.txt 2>&1; echo "rc=$?" >> gpurun_out/r2b_all.txt
timeout 300 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2b_c3.txt 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_sharded.py -q -p no:cacheprovider -x > gpurun_out/r2n_t.txt 2>&1; echo "rc=$?" >> gpurun_out/r2n_t.txt
timeout 300 python bench.py --workload c3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/r2n_c3.txt 2>&1
timeout 300 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r2n_c5.txt 2>&1

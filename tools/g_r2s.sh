mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_store.py tests/test_gpu_cas.py tests/test_gpu_exports.py -q -p no:cacheprovider -x > gpurun_out/r2s_t.txt 2>&1; echo "rc=$?" >> gpurun_out/r2s_t.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-extra > gpurun_out/r2s_c2.txt 2>&1

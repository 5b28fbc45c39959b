mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra > gpurun_out/r4f_c2.txt 2>&1
grep -h -o '"value": [0-9.]*\|"e2e": {"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r4f_c2.txt > gpurun_out/r4f_summary.txt
timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_store.py tests/test_gpu_reference_suite.py -q -m gpu -x > gpurun_out/r4f_t.txt 2>&1; echo rc=$? >> gpurun_out/r4f_t.txt

mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_store.py -q -m gpu -x > gpurun_out/r3h_t.txt 2>&1; echo rc=$? >> gpurun_out/r3h_t.txt
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r3h_c3.txt 2>&1
grep -h -o '"value": [0-9.]*\|"e2e": {"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r3h_c3.txt > gpurun_out/r3h_summary.txt
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_sharded.py -q -m gpu -x > gpurun_out/r3h_t2.txt 2>&1; echo rc=$? >> gpurun_out/r3h_t2.txt

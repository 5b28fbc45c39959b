mkdir -p gpurun_out
timeout 600 python bench.py --workload c2_01 --steps 3 --warmup 3 --no-cpu > gpurun_out/r4k_c201.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra > gpurun_out/r4k_c2.txt 2>&1
grep -h -o '"value": [0-9.]*\|"e2e": {"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r4k_c201.txt gpurun_out/r4k_c2.txt > gpurun_out/r4k_summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4k_launch.csv python bench.py --workload c2_01 --steps 1 --warmup 1 --no-cpu --no-e2e --batches 100 > gpurun_out/r4k_l.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_store.py tests/test_gpu_compat.py -q -m gpu -x > gpurun_out/r4k_t.txt 2>&1; echo rc=$? >> gpurun_out/r4k_t.txt

mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-e2e > gpurun_out/r4e_c2.txt 2>&1
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r4e_c3.txt 2>&1
grep -h -o '"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r4e_c2.txt gpurun_out/r4e_c3.txt > gpurun_out/r4e_summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4e_launch_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-extra --no-e2e --batches 100 > gpurun_out/r4e_l2.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_ndt.py -q -m gpu -x > gpurun_out/r4e_t.txt 2>&1; echo rc=$? >> gpurun_out/r4e_t.txt

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2z_t.txt 2>&1; echo rc=$? >> gpurun_out/r2z_t.txt
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2z_c3.txt 2>&1
grep -h -o '"value": [0-9.]*\|"e2e": {"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r2z_c3.txt > gpurun_out/r2z_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_ndt_det|k_nbk_fold" -c 2 -s 8 -o gpurun_out/r2z_ndt python tools/prof_run.py --workload c3 --batches 6 > gpurun_out/r2z_n.txt 2>&1

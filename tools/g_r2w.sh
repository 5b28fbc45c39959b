mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_store.py -x -q -m gpu > gpurun_out/r2w_t.txt 2>&1; echo rc=$? >> gpurun_out/r2w_t.txt
for v in 1 0; do
  if [ $v = 1 ]; then export VOXMAP_B200_NO_PIPELINE=1; else unset VOXMAP_B200_NO_PIPELINE; fi
  timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2w_c3_$v.txt 2>&1
done
grep -h -o '"value": [0-9.]*\|"e2e": {"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r2w_c3_*.txt > gpurun_out/r2w_summary.txt

mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2x_smoke.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_store.py tests/test_gpu_edges.py -x -q -m gpu > gpurun_out/r2x_t.txt 2>&1; echo rc=$? >> gpurun_out/r2x_t.txt
for v in 1 0; do
  if [ $v = 1 ]; then export VOXMAP_B200_NDT_GENERIC=1; else unset VOXMAP_B200_NDT_GENERIC; fi
  timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2x_c3_$v.txt 2>&1
done
grep -h -o '"value": [0-9.]*\|"e2e": {"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r2x_c3_*.txt > gpurun_out/r2x_summary.txt

mkdir -p gpurun_out
for v in main noagg main noagg; do
  if [ $v = main ]; then L=""; else L="libvoxmap_b200_$v.so"; fi
  VOXMAP_B200_LIB=$L timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-extra > gpurun_out/r2l_$v.txt 2>&1
  echo "$v $(grep -o '"value": [0-9.]*' gpurun_out/r2l_$v.txt | head -1) $(grep -o '"walk_ms": [0-9.]*' gpurun_out/r2l_$v.txt)" >> gpurun_out/r2l_summary.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_cas.py -q -p no:cacheprovider -x > gpurun_out/r2l_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2l_pytest.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det" -c 1 -s 5 -o gpurun_out/r2l_walk python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/r2l_ncu.txt 2>&1

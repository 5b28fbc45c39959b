mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_sharded.py -q -p no:cacheprovider -x > gpurun_out/r2p_t.txt 2>&1; echo "rc=$?" >> gpurun_out/r2p_t.txt
for v in main ndt3 ndt4 main; do
  if [ $v = main ]; then L=""; else L="libvoxmap_b200_$v.so"; fi
  VOXMAP_B200_LIB=$L timeout 300 python bench.py --workload c3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/r2p_$v.txt 2>&1
  echo "$v $(grep -o '"value": [0-9.]*' gpurun_out/r2p_$v.txt | head -1) $(grep -o '"stages_ms_per_step.*' gpurun_out/r2p_$v.txt)" >> gpurun_out/r2p_summary.txt
done

mkdir -p gpurun_out
for v in main b4c3 b3c3 main b4c3 b3c3; do
  if [ $v = main ]; then L=""; else L="libvoxmap_b200_$v.so"; fi
  VOXMAP_B200_LIB=$L timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-extra > gpurun_out/r2o_$v.txt 2>&1
  echo "$v $(grep -o '"value": [0-9.]*' gpurun_out/r2o_$v.txt | head -1) $(grep -o '"walk_ms": [0-9.]*' gpurun_out/r2o_$v.txt)" >> gpurun_out/r2o_summary.txt
done

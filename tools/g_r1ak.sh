mkdir -p gpurun_out
for v in main r2 r4b main r2 r4b; do
  if [ $v = main ]; then L=""; else L="libvoxmap_b200_$v.so"; fi
  VOXMAP_B200_LIB=$L timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ak_$v.txt 2>&1
  echo "$v $(grep -o '"value": [0-9.]*' gpurun_out/ak_$v.txt | head -1) $(grep -o '"resolve_ms": [0-9.]*' gpurun_out/ak_$v.txt)" >> gpurun_out/ak_summary.txt
done

mkdir -p gpurun_out
for v in main d3 main d3; do
  if [ $v = main ]; then L=""; else L="libvoxmap_b200_$v.so"; fi
  VOXMAP_B200_LIB=$L timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/at_$v.txt 2>&1
  echo "$v $(grep -o '"value": [0-9.]*' gpurun_out/at_$v.txt | head -1) $(grep -o '"discover_ms": [0-9.]*' gpurun_out/at_$v.txt)" >> gpurun_out/at_summary.txt
done

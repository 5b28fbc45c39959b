mkdir -p gpurun_out
for v in main f3 f4 main f3 f4; do
  if [ $v = main ]; then L=""; else L="libvoxmap_b200_$v.so"; fi
  VOXMAP_B200_LIB=$L timeout 600 python bench.py --workload c3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/aq_$v.txt 2>&1
  echo "$v $(grep -o '"value": [0-9.]*' gpurun_out/aq_$v.txt | head -1) $(grep -o '"fold_ms": [0-9.]*' gpurun_out/aq_$v.txt)" >> gpurun_out/aq_summary.txt
done

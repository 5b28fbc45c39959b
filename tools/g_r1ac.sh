mkdir -p gpurun_out
for v in g1k g512 g256 g64 g1k g256 g64; do
  L="libvoxmap_b200_$v.so"
  VOXMAP_B200_LIB=$L timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ac_$v.txt 2>&1
  echo "$v $(grep -o '"value": [0-9.]*' gpurun_out/ac_$v.txt | head -1) $(grep -o '"walk_ms": [0-9.]*' gpurun_out/ac_$v.txt)" >> gpurun_out/ac_summary.txt
done
VOXMAP_B200_LIB=libvoxmap_b200_g64.so timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ac_c1_g64.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_g1k.so timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ac_c1_g1k.txt 2>&1

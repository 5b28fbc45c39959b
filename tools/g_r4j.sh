mkdir -p gpurun_out
for v in big1 base big8; do
  if [ $v = base ]; then unset VOXMAP_B200_LIB; else export VOXMAP_B200_LIB=libvoxmap_b200_$v.so; fi
  timeout 600 python bench.py --workload c2_01 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r4j_$v.txt 2>&1
  echo $v $(grep -h -o '"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r4j_$v.txt | head -2) >> gpurun_out/r4j_summary.txt
done

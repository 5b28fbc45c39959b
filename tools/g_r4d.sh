mkdir -p gpurun_out
for v in base rp rp4 rp6; do
  if [ $v = base ]; then unset VOXMAP_B200_LIB; else export VOXMAP_B200_LIB=libvoxmap_b200_$v.so; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-e2e > gpurun_out/r4d_$v.txt 2>&1
  echo $v $(grep -h -o '"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r4d_$v.txt | head -2) >> gpurun_out/r4d_summary.txt
done

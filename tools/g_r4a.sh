mkdir -p gpurun_out
for v in base ncb3; do
  if [ $v = base ]; then unset VOXMAP_B200_LIB; else export VOXMAP_B200_LIB=libvoxmap_b200_$v.so; fi
  timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r4a_$v.txt 2>&1
  echo $v $(grep -h -o '"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r4a_$v.txt | head -2) >> gpurun_out/r4a_summary.txt
done
unset VOXMAP_B200_LIB
timeout 900 python -m pytest tests/test_gpu_ndt.py -q -m gpu -x > gpurun_out/r4a_t.txt 2>&1; echo rc=$? >> gpurun_out/r4a_t.txt

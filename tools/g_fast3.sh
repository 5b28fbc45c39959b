# verified fast operators in the three-lane NDT fold: parity, C3 A/B against the IEEE-only build, slowest task
mkdir -p gpurun_out
T=x3
timeout 1500 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -q > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
for i in 1 2; do
timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c3_fast_$i.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_ieee.so timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c3_ieee_$i.txt 2>&1
done
VOXMAP_B200_LIB=libvoxmap_b200_prof.so timeout 300 python tools/prof_run.py --workload c3 --batches 6 > gpurun_out/${T}_prof.txt 2>&1

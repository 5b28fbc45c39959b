# verified fast divisions in the occupancy hit step: parity, C2@0.1 m and C2 A/B against IEEE-only
mkdir -p gpurun_out
T=bx
timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -q -x > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
for i in 1 2; do
timeout 600 python bench.py --workload c2_01 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c201_fast_$i.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_ieee.so timeout 600 python bench.py --workload c2_01 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c201_ieee_$i.txt 2>&1
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/${T}_c2_fast.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_ieee.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/${T}_c2_ieee.txt 2>&1

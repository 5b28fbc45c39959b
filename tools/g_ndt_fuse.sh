# NDT bucket preparation fused (4 launches) vs split (10): parity, C3 A/B, launch lists
mkdir -p gpurun_out
T=nf
timeout 1200 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_sharded.py tests/test_gpu_parity.py -q > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
for i in 1 2; do
timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c3_fused_$i.txt 2>&1
VOXMAP_B200_NBK_SPLIT=1 timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c3_split_$i.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_c3.csv python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_l3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_c201.csv python bench.py --workload c2_01 --steps 1 --warmup 1 --no-cpu --no-e2e --batches 100 > gpurun_out/${T}_l201.txt 2>&1

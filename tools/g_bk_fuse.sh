# occupancy folds in one launch (block roles) vs three: parity, C2 / C2@0.1m A/B
mkdir -p gpurun_out
T=bf
timeout 1500 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_store.py tests/test_gpu_compat.py -q -x > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
for i in 1 2; do
timeout 600 python bench.py --workload c2_01 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c201_fused_$i.txt 2>&1
VOXMAP_B200_BK_SPLIT=1 timeout 600 python bench.py --workload c2_01 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c201_split_$i.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/${T}_c2_fused_$i.txt 2>&1
VOXMAP_B200_BK_SPLIT=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-extra > gpurun_out/${T}_c2_split_$i.txt 2>&1
done

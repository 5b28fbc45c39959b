# NDT fold with three lanes per bucket (rotations pipelined) vs one lane: parity, C3 A/B; sharded suite (merged syncs)
mkdir -p gpurun_out
T=f3
timeout 1500 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
for i in 1 2; do
timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c3_new_$i.txt 2>&1
VOXMAP_B200_FOLD1=1 timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c3_old_$i.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_c3.csv python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_l3.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det|k_bk_fold_all" -s 20 -c 2 -o gpurun_out/${T}_full_c2 python tools/prof_run.py --workload c2 --batches 20 > gpurun_out/${T}_ncu2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_nbk_fold3" -s 10 -c 1 -o gpurun_out/${T}_full_fold3 python tools/prof_run.py --workload c3 --batches 20 > gpurun_out/${T}_ncu3.txt 2>&1

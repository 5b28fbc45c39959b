mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4h_launch.csv python bench.py --workload c2_01 --steps 1 --warmup 1 --no-cpu --no-e2e --batches 100 > gpurun_out/r4h_l.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bk_fold" -c 2 -s 20 -o gpurun_out/r4h_fold python tools/prof_run.py --workload c2_01 --batches 300 --device > gpurun_out/r4h_n.txt 2>&1
VOXMAP_B200_NDT_DEBUG=1 timeout 300 python tools/prof_run.py --workload c2_01 --batches 100 > gpurun_out/r4h_dbg.txt 2>&1

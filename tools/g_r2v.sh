mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v_launch_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra --batches 100 > gpurun_out/r2v_l.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det" -c 1 -s 10 -o gpurun_out/r2v_walk_c2 python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/r2v_n1.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_ndt|k_nbk_fold" -c 2 -s 8 -o gpurun_out/r2v_ndt_c3 python tools/prof_run.py --workload c3 --batches 6 > gpurun_out/r2v_n2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v_launch_c3.csv python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r2v_l3.txt 2>&1

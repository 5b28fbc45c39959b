mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det|k_discover|k_resolve|k_bk_fold" -s 16 -c 4 -o gpurun_out/as_full_c2 python tools/prof_run.py --workload c2 --batches 100 --device > gpurun_out/as_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_ndt|k_fold_ndt" -s 4 -c 2 -o gpurun_out/as_full_c3 python tools/prof_run.py --workload c3 --batches 6 --device > gpurun_out/as_ncu3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/as_launches_c2.csv python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/as_launch.txt 2>&1

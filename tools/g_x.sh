mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fold_ndt" -s 5 -c 1 -o gpurun_out/x_prof_c3 python tools/prof_run.py --workload c3 --batches 20 > gpurun_out/x_ncu_c3.txt 2>&1

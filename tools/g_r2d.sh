mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_nbk|k_walk_ndt" -s 16 -c 8 -o gpurun_out/r2d_ndt python tools/prof_run.py --workload c3 --batches 5 > gpurun_out/r2d_ncu.txt 2>&1

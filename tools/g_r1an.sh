mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_ndt|k_fold_ndt|k_resolve|k_discover" -s 8 -c 4 -o gpurun_out/an_full_c3 python tools/prof_run.py --workload c3 --batches 6 --device > gpurun_out/an_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_bk_fold|k_bk_scatter|k_bk_count" -s 6 -c 3 -o gpurun_out/an_full_bk python tools/prof_run.py --workload c2 --batches 60 --device > gpurun_out/an_ncu2.txt 2>&1

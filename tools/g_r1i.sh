mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det|k_discover|k_resolve" -s 12 -c 3 -o gpurun_out/i_prof_c2 python tools/prof_run.py --workload c2 --batches 100 --device > gpurun_out/i_ncu.txt 2>&1

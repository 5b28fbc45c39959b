mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det|k_discover|k_resolve" -c 3 -s 15 -o gpurun_out/r2m_c2 python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/r2m_ncu.txt 2>&1

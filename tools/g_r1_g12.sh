mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/g12_c2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_resolve|k_discover|k_walk" -s 6 -c 3 -o gpurun_out/prof12_c2 python tools/prof_run.py --workload c2 --batches 60 > gpurun_out/g12_ncu.txt 2>&1

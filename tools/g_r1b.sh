mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/b_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/b_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk|k_resolve|k_discover" -s 30 -c 3 -o gpurun_out/b_prof_c2 python tools/prof_run.py --workload c2 --batches 300 > gpurun_out/b_ncu.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk" -s 10 -c 1 -o gpurun_out/b_prof_c2cas python tools/prof_run.py --workload c2 --exec cas --batches 300 > gpurun_out/b_ncu_cas.txt 2>&1

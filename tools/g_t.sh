mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/t_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --batches 1000 > gpurun_out/t_launch_run.txt 2>&1
bash tools/g_prof.sh t
bash tools/g_prof_all.sh t
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fold_ndt|k_walk_ndt" -s 20 -c 2 -o gpurun_out/t_prof_c3 python tools/prof_run.py --workload c3 --batches 10 > gpurun_out/t_ncu_c3.txt 2>&1

mkdir -p gpurun_out
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/fb_bench.txt 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fb_ref.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fb_launch_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-extra --no-e2e --batches 100 > gpurun_out/fb_l2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fb_launch_c3.csv python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/fb_l3.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det|k_resolve" -c 2 -s 20 -o gpurun_out/fb_c2 python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/fb_n1.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_ndt_det|k_nbk_fold" -c 2 -s 16 -o gpurun_out/fb_c3 python tools/prof_run.py --workload c3 --batches 20 > gpurun_out/fb_n2.txt 2>&1

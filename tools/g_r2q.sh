mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -p no:cacheprovider -k "tsdf or c4 or golden or degenerate or hot" > gpurun_out/r2q_t.txt 2>&1; echo "rc=$?" >> gpurun_out/r2q_t.txt
timeout 300 python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu --no-e2e --batches 20 > gpurun_out/r2q_c4.txt 2>&1
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-extra > gpurun_out/r2q_c2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_ndt|k_ndt_weigh" -c 2 -s 8 -o gpurun_out/r2q_ndt python tools/prof_run.py --workload c3 --batches 6 > gpurun_out/r2q_ncu.txt 2>&1

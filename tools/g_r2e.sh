mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ndt.py -q -x -p no:cacheprovider > gpurun_out/r2e_ndt.txt 2>&1; echo "rc=$?" >> gpurun_out/r2e_ndt.txt
timeout 300 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2e_c3.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_nbk" -s 16 -c 9 -o gpurun_out/r2e_ndt python tools/prof_run.py --workload c3 --batches 5 > gpurun_out/r2e_ncu.txt 2>&1

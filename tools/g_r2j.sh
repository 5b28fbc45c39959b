mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_store.py tests/test_cli.py -q -p no:cacheprovider > gpurun_out/r2j_store.txt 2>&1; echo "rc=$?" >> gpurun_out/r2j_store.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det" -c 1 -s 10 -o gpurun_out/r2j_walk python tools/prof_run.py --workload c2 --batches 30 --device > gpurun_out/r2j_ncu1.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_discover" -c 1 -s 10 -o gpurun_out/r2j_disc python tools/prof_run.py --workload c2 --batches 30 --device > gpurun_out/r2j_ncu2.txt 2>&1

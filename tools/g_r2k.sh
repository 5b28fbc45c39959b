mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2k_launch.csv python tools/prof_run.py --workload c2 --batches 3 --device > gpurun_out/r2k_l.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_reference_suite.py tests/test_cli.py -q -p no:cacheprovider > gpurun_out/r2k_ref.txt 2>&1; echo "rc=$?" >> gpurun_out/r2k_ref.txt

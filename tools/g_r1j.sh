mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q > gpurun_out/j_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/j_pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/j_c2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/j_launches_c2.csv python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/j_launch.txt 2>&1

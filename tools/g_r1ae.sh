mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/ae_c2.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --exec cas > gpurun_out/ae_c2cas.txt 2>&1
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/ae_c1.txt 2>&1
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/ae_c3.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ae_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/ae_pytest_all.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ae_launches_c2.csv python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/ae_launch.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det|k_discover|k_resolve" -s 18 -c 3 -o gpurun_out/ae_full_c2 python tools/prof_run.py --workload c2 --batches 100 --device > gpurun_out/ae_ncu.txt 2>&1

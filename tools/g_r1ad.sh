mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ad_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/ad_pytest_all.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ad_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/ad_smoke.txt
timeout 900 python bench.py > gpurun_out/ad_c2.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --exec cas > gpurun_out/ad_c2cas.txt 2>&1
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/ad_c1.txt 2>&1
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/ad_c3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ad_launches_c2.csv python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/ad_launch.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det|k_discover" -s 12 -c 2 -o gpurun_out/ad_full_c2 python tools/prof_run.py --workload c2 --batches 100 --device > gpurun_out/ad_ncu.txt 2>&1

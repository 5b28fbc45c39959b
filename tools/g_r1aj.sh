mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/aj_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/aj_pytest_all.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/aj_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/aj_smoke.txt
timeout 900 python bench.py > gpurun_out/aj_c2.txt 2>&1
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/aj_c3.txt 2>&1
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/aj_c1.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --exec cas > gpurun_out/aj_c2cas.txt 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/aj_ref.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/aj_launches_c3.csv python tools/prof_run.py --workload c3 --batches 6 --device > gpurun_out/aj_launch3.txt 2>&1

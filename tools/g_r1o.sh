mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/o_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/o_pytest_all.txt
timeout 900 python bench.py > gpurun_out/o_c2.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/o_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/o_smoke.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/o_launches_c2.csv python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/o_launch.txt 2>&1

mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/h_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/h_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/h_smoke.txt
timeout 900 python bench.py > gpurun_out/h_c2.txt 2>&1
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/h_c1.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --exec cas > gpurun_out/h_c2cas.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/h_ref.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/h_launches_c2.csv python tools/prof_run.py --workload c2 --batches 100 > gpurun_out/h_launch.txt 2>&1

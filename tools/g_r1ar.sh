mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ar_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/ar_pytest_all.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ar_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/ar_smoke.txt
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/ar_c3.txt 2>&1
timeout 900 python bench.py > gpurun_out/ar_c2.txt 2>&1

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s -k "cas_order_free or not slow" > gpurun_out/ag_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/ag_pytest.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ag_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/ag_pytest_all.txt
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/ag_c1.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ag_c2.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ag_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/ag_smoke.txt

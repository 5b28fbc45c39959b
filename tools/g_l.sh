mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/l_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/l_pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/l_c2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_discover|k_resolve|k_seg" -s 40 -c 4 -o gpurun_out/l_prof python tools/prof_run.py --workload c2 --batches 300 > gpurun_out/l_ncu.txt 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/m_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/m_pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/m_c2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/m_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/m_pytest_all.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_discover" -s 12 -c 1 -o gpurun_out/m_prof_disc python tools/prof_run.py --workload c2 --batches 100 --device > gpurun_out/m_ncu.txt 2>&1

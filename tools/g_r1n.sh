mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/n_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/n_pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/n_c2.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_resu.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/n_c2_resu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/n_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/n_pytest_all.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_discover" -s 12 -c 1 -o gpurun_out/n_prof_disc python tools/prof_run.py --workload c2 --batches 100 --device > gpurun_out/n_ncu.txt 2>&1

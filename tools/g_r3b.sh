mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_store.py -q -m gpu -x > gpurun_out/r3b_t.txt 2>&1; echo rc=$? >> gpurun_out/r3b_t.txt
VOXMAP_B200_LIB=libvoxmap_b200_nodefer.so timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-e2e > gpurun_out/r3b_c2_0.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra > gpurun_out/r3b_c2_1.txt 2>&1
grep -h -o '"value": [0-9.]*\|"e2e": {"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r3b_c2_0.txt gpurun_out/r3b_c2_1.txt > gpurun_out/r3b_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det" -c 1 -s 10 -o gpurun_out/r3b_walk python tools/prof_run.py --workload c2 --batches 300 --device > gpurun_out/r3b_n.txt 2>&1

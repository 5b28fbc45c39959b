mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "arith or hypot or division" > gpurun_out/r3e_t0.txt 2>&1; echo rc=$? >> gpurun_out/r3e_t0.txt
VOXMAP_B200_LIB=libvoxmap_b200_foldprof.so timeout 300 python tools/prof_run.py --workload c3 --batches 6 > gpurun_out/r3e_fold.txt 2>&1
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r3e_c3.txt 2>&1
grep -h -o '"value": [0-9.]*\|"e2e": {"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r3e_c3.txt > gpurun_out/r3e_summary.txt
timeout 1200 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_sharded.py -q -m gpu -x > gpurun_out/r3e_t.txt 2>&1; echo rc=$? >> gpurun_out/r3e_t.txt

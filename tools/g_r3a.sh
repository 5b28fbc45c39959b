mkdir -p gpurun_out
VOXMAP_B200_LIB=libvoxmap_b200_foldprof.so timeout 300 python tools/prof_run.py --workload c3 --batches 12 > gpurun_out/r3a_fold.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q -m gpu -x > gpurun_out/r3a_t.txt 2>&1; echo rc=$? >> gpurun_out/r3a_t.txt
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r3a_c3.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra > gpurun_out/r3a_c2.txt 2>&1
grep -h -o '"value": [0-9.]*\|"e2e": {"value": [0-9.]*\|stages_ms_per_step[^}]*' gpurun_out/r3a_c3.txt gpurun_out/r3a_c2.txt > gpurun_out/r3a_summary.txt

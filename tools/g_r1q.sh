mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_edges.py -q -k "fold_paths" > gpurun_out/q_t1.txt 2>&1; echo "rc=$?" >> gpurun_out/q_t1.txt
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_edges.py -x -q -k "fold_paths" > gpurun_out/q_san.txt 2>&1; echo "rc=$?" >> gpurun_out/q_san.txt
timeout 300 python -m pytest tests/test_gpu_edges.py -x -q -k "overflow" > gpurun_out/q_t2.txt 2>&1; echo "rc=$?" >> gpurun_out/q_t2.txt

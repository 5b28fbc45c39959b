mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_edges.py -x -q -k "block-large" > gpurun_out/p_t1.txt 2>&1; echo "rc=$?" >> gpurun_out/p_t1.txt
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_edges.py -x -q -k "block-large" > gpurun_out/p_san.txt 2>&1; echo "rc=$?" >> gpurun_out/p_san.txt
timeout 300 python -m pytest tests/test_gpu_edges.py -x -q -k "overflow" > gpurun_out/p_t2.txt 2>&1; echo "rc=$?" >> gpurun_out/p_t2.txt

mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_edges.py -q -p no:cacheprovider -x -k "fold_paths and thread" > gpurun_out/r2t_san.txt 2>&1

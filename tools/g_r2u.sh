mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -q -p no:cacheprovider -x -k "record_overflow or pool_replays" > gpurun_out/r2u_t.txt 2>&1; echo "rc=$?" >> gpurun_out/r2u_t.txt

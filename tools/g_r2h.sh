mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sharded.py -q -x -p no:cacheprovider -k ndt > gpurun_out/r2h_shard.txt 2>&1; echo "rc=$?" >> gpurun_out/r2h_shard.txt
timeout 1200 python -m pytest tests/test_gpu_edges.py -q -p no:cacheprovider -k "c4 or c5 or twenty" > gpurun_out/r2h_edges.txt 2>&1; echo "rc=$?" >> gpurun_out/r2h_edges.txt
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -p no:cacheprovider -k "not ndt" > gpurun_out/r2h_shard_occ.txt 2>&1; echo "rc=$?" >> gpurun_out/r2h_shard_occ.txt

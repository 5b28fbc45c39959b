mkdir -p gpurun_out
timeout 600 python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu --batches 20 > gpurun_out/r2i_c4.txt 2>&1
timeout 600 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu > gpurun_out/r2i_c5.txt 2>&1
VM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload c3 --steps 1 --warmup 1 --no-e2e > gpurun_out/r2i_shard_c3.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det|k_discover" -s 20 -c 2 -o gpurun_out/r2i_c2 python tools/prof_run.py --workload c2 --batches 30 --device > gpurun_out/r2i_ncu.txt 2>&1

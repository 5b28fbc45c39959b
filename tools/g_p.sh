mkdir -p gpurun_out
VM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 1 --warmup 1 --batches 200 > gpurun_out/p_shard2.txt 2>&1
tail -c 3000 gpurun_out/p_shard2.txt

mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/r_base.txt 2>&1
bash tools/g_prof.sh r
cp paper_2206_06079_b200/_lib/libvoxmap_b200.so /tmp/keep.so
cp gpurun_v4.so paper_2206_06079_b200/_lib/libvoxmap_b200.so
timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/r_v4.txt 2>&1

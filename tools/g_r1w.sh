mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/w_c2.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_k2.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/w_c2_k2.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_k4.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/w_c2_k4.txt 2>&1

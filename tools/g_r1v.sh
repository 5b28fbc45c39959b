mkdir -p gpurun_out
VOXMAP_B200_LIB=libvoxmap_b200_d512.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/v_c2_d512.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_d1024.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/v_c2_d1024.txt 2>&1

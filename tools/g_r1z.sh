mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/z_c2.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_c16.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/z_c2_c16.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_c16.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "not ndt" > gpurun_out/z_pytest_c16.txt 2>&1; echo "rc=$?" >> gpurun_out/z_pytest_c16.txt

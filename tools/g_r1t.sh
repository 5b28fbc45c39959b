mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/t_pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/t_c2.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_r4.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/t_c2_r4.txt 2>&1

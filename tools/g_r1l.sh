mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/l_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/l_pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/l_c2.txt 2>&1
VOXMAP_B200_LIB=libvoxmap_b200_bmg.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/l_c2_bmg.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/l_c2b.txt 2>&1

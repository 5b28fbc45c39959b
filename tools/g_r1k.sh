mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/k_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/k_pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/k_c2.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --per-batch > gpurun_out/k_c2pb.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/k_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/k_pytest_all.txt

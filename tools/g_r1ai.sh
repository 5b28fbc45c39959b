mkdir -p gpurun_out
timeout 600 python bench.py --workload c3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ai_c3.txt 2>&1
VOXMAP_B200_NO_RAY_ORDER=1 timeout 600 python bench.py --workload c3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ai_c3_noro.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ndt or NDT or golden or tunnel" > gpurun_out/ai_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/ai_pytest.txt

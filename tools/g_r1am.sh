mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider -k "prefetched or submit_batches" > gpurun_out/am_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/am_pytest.txt
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/am_c3.txt 2>&1
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --per-batch > gpurun_out/am_c3pb.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/am_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/am_pytest_all.txt

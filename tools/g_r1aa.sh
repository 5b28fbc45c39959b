mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/aa_c2.txt 2>&1
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/aa_c1.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --exec cas > gpurun_out/aa_c2cas.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/aa_pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/aa_pytest_all.txt

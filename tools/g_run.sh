# usage: bash tools/g_run.sh TAG -- tests + C1/C2 benches + ncu of the C2 walk
T=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.txt
timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c1.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_c2.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --exec cas > gpurun_out/${T}_c2cas.txt 2>&1
bash tools/g_prof.sh $T

# round-end evidence (tag $1): smoke, the whole GPU suite, default bench, reference arm, launch lists, ncu of the NDT fold
T=${1:-k}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
timeout 900 python bench.py > gpurun_out/${T}_bench.txt 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra --batches 200 > gpurun_out/${T}_l2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_c3.csv python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_l3.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_nbk_fold3|k_walk_det" -s 10 -c 2 -o gpurun_out/${T}_full_fold3 python tools/prof_run.py --workload c3 --batches 20 > gpurun_out/${T}_ncu3.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det" -s 10 -c 1 -o gpurun_out/${T}_full_walk python tools/prof_run.py --workload c2 --batches 300 > gpurun_out/${T}_ncu2.txt 2>&1

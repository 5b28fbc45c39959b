# round evidence (tag $1): default bench line, reference arm, launch lists, ncu --set full of the top kernels
T=${1:-h}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
timeout 900 python bench.py > gpurun_out/${T}_bench.txt 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra --batches 200 > gpurun_out/${T}_l2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_c3.csv python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_l3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_c201.csv python bench.py --workload c2_01 --steps 1 --warmup 1 --no-cpu --no-e2e --batches 200 > gpurun_out/${T}_l201.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_det|k_bk_fold_all|k_resolve|k_discover" -s 40 -c 4 -o gpurun_out/${T}_full_c2 python tools/prof_run.py --workload c2 --batches 300 > gpurun_out/${T}_ncu2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_ndt_det|k_nbk_fold3|k_nbk_sort_gather|k_nbk_weigh_count" -s 40 -c 4 -o gpurun_out/${T}_full_c3 python tools/prof_run.py --workload c3 --batches 20 > gpurun_out/${T}_ncu3.txt 2>&1
ls -la gpurun_out/ > gpurun_out/${T}_ls.txt

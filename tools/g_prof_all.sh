# ncu --set full of one launch of every kernel of a C2 batch (after warm-up)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_discover|k_resolve|k_fold|k_seg|k_rgrid|Onesweep" -s 60 -c 9 -o gpurun_out/$1_prof_all python tools/prof_run.py --workload c2 --batches 300 > gpurun_out/$1_ncu_all.txt 2>&1

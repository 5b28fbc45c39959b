# usage: bash tools/g_prof.sh TAG [exec]   -- ncu --set full of one walk launch of C2
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_walk" -s 10 -c 1 -o gpurun_out/$1_prof_c2 python tools/prof_run.py --workload c2 --batches 300 --exec ${2:-det} > gpurun_out/$1_ncu.txt 2>&1

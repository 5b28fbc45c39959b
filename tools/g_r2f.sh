mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ndt.py -q -x -p no:cacheprovider > gpurun_out/r2f_ndt.txt 2>&1; echo "rc=$?" >> gpurun_out/r2f_ndt.txt
timeout 300 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2f_c3.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_nbk_fold|k_nbk_gather|k_nbk_sort_small" -s 6 -c 3 -o gpurun_out/r2f_ndt python tools/prof_run.py --workload c3 --batches 5 > gpurun_out/r2f_ncu.txt 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2206_06079_b200 import _native
for fp in (16<<20, 64<<20, 256<<20, 1<<30):
    print(fp, _native.probe_red_rate(0, fp, 5))
" > gpurun_out/r2f_red.txt 2>&1

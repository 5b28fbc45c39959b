# straight-line hypot: parity, C3 bench; slowest fold task (VM_FOLD_PROF dev build), three-lane vs one-lane fold
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ndt.py -q > gpurun_out/p3_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/p3_tests.txt
for i in 1 2; do
timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/p3_c3_$i.txt 2>&1
done
VOXMAP_B200_LIB=libvoxmap_b200_prof.so timeout 300 python tools/prof_run.py --workload c3 --batches 12 > gpurun_out/p3_new.txt 2>&1
VOXMAP_B200_FOLD1=1 VOXMAP_B200_LIB=libvoxmap_b200_prof.so timeout 300 python tools/prof_run.py --workload c3 --batches 12 > gpurun_out/p3_old.txt 2>&1

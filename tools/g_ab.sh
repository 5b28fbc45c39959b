# A/B runs behind DESIGN's "Launch fusion" and "Tried and rejected" rows (on the GPU box):
#   bash tools/g_ab.sh nbk     NDT bucket preparation: 4 launches vs 10 (VOXMAP_B200_NBK_SPLIT=1)
#   bash tools/g_ab.sh bk      occupancy folds: 1 launch vs 3 (VOXMAP_B200_BK_SPLIT=1)
#   bash tools/g_ab.sh fold3   NDT fold: three lanes per voxel vs one (VOXMAP_B200_FOLD1=1)
#   bash tools/g_ab.sh fast    verified branch-free division in both folds (variant build NBK3_FAST=1 BK_FAST=1)
# each: the parity suites of the path first, then two bench runs per arm into gpurun_out/ab_*
mkdir -p gpurun_out
case "$1" in
  nbk)   W=c3;    ENV=VOXMAP_B200_NBK_SPLIT=1; SUITES="tests/test_gpu_ndt.py tests/test_gpu_sharded.py" ;;
  bk)    W=c2_01; ENV=VOXMAP_B200_BK_SPLIT=1;  SUITES="tests/test_gpu_edges.py tests/test_gpu_parity.py" ;;
  fold3) W=c3;    ENV=VOXMAP_B200_FOLD1=1;     SUITES="tests/test_gpu_ndt.py tests/test_gpu_parity.py" ;;
  fast)  W=c3;    SUITES="tests/test_gpu_ndt.py tests/test_gpu_edges.py"
         python -c "from paper_2206_06079_b200 import _build; _build.build_variant('libvoxmap_b200_fast.so', ['NBK3_FAST=1', 'BK_FAST=1'])"
         ENV=VOXMAP_B200_LIB=libvoxmap_b200_fast.so ;;
  *) echo "usage: $0 nbk|bk|fold3|fast"; exit 2 ;;
esac
timeout 1500 python -m pytest $SUITES -q > gpurun_out/ab_$1_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/ab_$1_tests.txt
for i in 1 2; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_$1_default_$i.txt 2>&1
  env $ENV timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_$1_other_$i.txt 2>&1
done

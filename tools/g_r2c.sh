mkdir -p gpurun_out
cat > /tmp/dbg.py <<'PY'
import sys; sys.path.insert(0,'.')
from paper_2206_06079_b200 import scans, MapConfig, VoxelMap, submit_batch, ExecutorOptions
from paper_2206_06079_b200.layers import MODE_LAYERS
d=scans.os64_tunnel_scans(6)
vm=VoxelMap(MapConfig(), MODE_LAYERS['ndt-om'])
for b in d:
    st=submit_batch(vm,b,'ndt-om')
    print(st.gpu_time*1e3, st.walk_time*1e3, st.records, st.marked_voxels, file=sys.stderr)
PY
VOXMAP_B200_NDT_DEBUG=1 timeout 300 python /tmp/dbg.py > gpurun_out/r2c_dbg.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ndt.py tests/test_gpu_cas.py tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/r2c_t.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c_t.txt

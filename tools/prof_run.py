"""Short driver for ncu captures: integrate a few batches of a workload."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2206_06079_b200 import ExecutorOptions, MapConfig, VoxelMap, scans, submit_batch  # noqa
from paper_2206_06079_b200.layers import MODE_LAYERS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c1")
ap.add_argument("--exec", dest="exec_", default="det")
ap.add_argument("--batches", type=int, default=4)
a = ap.parse_args()
if a.workload == "c1":
    cfg, mode, data = MapConfig(), "occupancy", [scans.os64_room_scan()] * a.batches
elif a.workload == "c2":
    cfg, mode = MapConfig(voxel_size=0.05), "occupancy"
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(a.batches)))
else:
    cfg, mode, data = MapConfig(), "ndt-om", scans.os64_tunnel_scans(a.batches)
vm = VoxelMap(cfg, MODE_LAYERS[mode], initial_regions=4096)
for b in data:
    st = submit_batch(vm, b, mode, ExecutorOptions(deterministic=a.exec_ == "det"))
print(st)

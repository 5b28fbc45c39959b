"""Short driver for ncu captures: integrate a few batches of a workload.

--device keeps the records in HBM (the bench's `value` path: one discover
launch per batch); without it batches go through submit_batch from host
records (the `e2e` path: chunked upload + discover).
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2206_06079_b200 import ExecutorOptions, MapConfig, VoxelMap, scans, submit_batch  # noqa
from paper_2206_06079_b200 import _native  # noqa: E402
from paper_2206_06079_b200.layers import MODE_LAYERS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c1")
ap.add_argument("--exec", dest="exec_", default="det")
ap.add_argument("--batches", type=int, default=4)
ap.add_argument("--device", action="store_true")
a = ap.parse_args()
if a.workload == "c1":
    cfg, mode, data = MapConfig(), "occupancy", [scans.os64_room_scan()] * a.batches
elif a.workload in ("c2", "c2_01"):
    cfg, mode = MapConfig(voxel_size=0.05 if a.workload == "c2" else 0.1), "occupancy"
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(a.batches)))
else:
    cfg, mode, data = MapConfig(), "ndt-om", scans.os64_tunnel_scans(a.batches)
vm = VoxelMap(cfg, MODE_LAYERS[mode], initial_regions=4096)
if a.device:
    import torch
    host = np.concatenate(data)
    sizes = [len(b) for b in data]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    d_rec = torch.from_numpy(host.view(np.uint8).copy()).to("cuda:0")
    torch.cuda.synchronize()
    vm._native.set_stream(torch.cuda.current_stream().cuda_stream)
    for b in range(len(data)):
        r = _native.rays_from_records(sizes[b], d_rec.data_ptr() + int(offs[b]) * 40)
        st = vm._native.integrate(r, mode, a.exec_ == "det")
    torch.cuda.synchronize()
else:
    for b in data:
        st = submit_batch(vm, b, mode, ExecutorOptions(deterministic=a.exec_ == "det"))
print(st)

"""TSDF query (mirror of voxmap.tsdf, tsdf.py:29-34); the merge runs on the device."""
from __future__ import annotations

from .keys import key_for_point


def tsdf_query(vmap, point):
    values = vmap.voxel_values("tsdf", key_for_point(point, vmap.cfg))
    if values is None or values[1] == 0.0:
        return None
    return float(values[0]), float(values[1])

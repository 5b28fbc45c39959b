"""Ray record, preprocessing helpers and the (GPU) voxel walk.

Mirror of voxmap.traversal (traversal.py:20-178).  `clip_ray` and
`segment_ray` are the per-ray API helpers; the batch path performs the
same arithmetic on the device (csrc/vm_device.cuh: prep_ray / segment_of).
`walk_voxels*` run the CUDA DDA (vm_walk_voxels), bit-identical to the
reference walk.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import NamedTuple

import numpy as np

from . import _native
from .keys import VoxelKey, key_for_global


@dataclass(frozen=True)
class RaySample:
    """One sensor ray (traversal.py:20-42)."""

    origin: np.ndarray
    end: np.ndarray
    intensity: float = 0.0
    has_sample: bool = True
    timestamp: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "origin", np.asarray(self.origin, dtype=np.float64))
        object.__setattr__(self, "end", np.asarray(self.end, dtype=np.float64))
        if not (np.all(np.isfinite(self.origin)) and np.all(np.isfinite(self.end))):
            raise ValueError("ray endpoints must be finite")

    @property
    def length(self) -> float:
        return float(np.linalg.norm(self.end - self.origin))


class VoxelVisit(NamedTuple):
    key: VoxelKey
    entry_t: float
    exit_t: float
    path_length: float


def _walk_cap(origin, end, cell: float) -> int:
    return sum(abs(math.floor(float(end[a]) / cell) - math.floor(float(origin[a]) / cell))
               for a in range(3)) + 2


def _walk(origin, end, cell: float):
    o = [float(c) for c in origin]
    e = [float(c) for c in end]
    return _native.walk_voxels_native(*o, *e, cell) if _walk_cap(o, e, cell) <= 4096 else \
        _walk_big(o, e, cell)


def _walk_big(o, e, cell):
    import ctypes
    cap = _walk_cap(o, e, cell)
    coords = np.empty((cap, 3), dtype=np.int64)
    t0 = np.empty(cap)
    t1 = np.empty(cap)
    n = ctypes.c_int64()
    _native.check(_native.lib().vm_walk_voxels(*o, *e, float(cell), cap,
                                                coords.ctypes.data_as(ctypes.c_void_p),
                                                t0.ctypes.data_as(ctypes.c_void_p),
                                                t1.ctypes.data_as(ctypes.c_void_p),
                                                ctypes.byref(n)), "vm_walk_voxels")
    k = int(n.value)
    return coords[:k], t0[:k], t1[:k]


def walk_voxels_global(origin, end, cfg):
    """(global coords [n,3] int64, entry_t, exit_t) -- traversal.py:124-131."""
    return _walk(origin, end, cfg.voxel_size)


def walk_voxels(ray: RaySample, cfg) -> list[VoxelVisit]:
    coords, t0, t1 = _walk(ray.origin, ray.end, cfg.voxel_size)
    length = ray.length
    return [VoxelVisit(key_for_global(c, cfg), float(a), float(b), float((b - a) * length))
            for c, a, b in zip(coords, t0, t1)]


def walk_regions(ray: RaySample, cfg) -> list[tuple[int, int, int]]:
    coords, _, _ = _walk(ray.origin, ray.end, cfg.region_size)
    return [tuple(int(x) for x in c) for c in coords]


def clip_ray(ray: RaySample, cfg) -> RaySample:
    """traversal.py:140-150: a ray longer than max_ray_range is cut to it and
    keeps no sample (miss evidence only)."""
    length = ray.length
    if length > cfg.max_ray_range:
        unit = (ray.end - ray.origin) / length
        ray = replace(ray, end=ray.origin + unit * cfg.max_ray_range, has_sample=False)
    return ray


def segment_ray(ray: RaySample, cfg) -> list[RaySample]:
    """traversal.py:153-178: pieces of at most segment_length along the ray;
    the last piece ends exactly at ray.end and alone keeps has_sample.  (The
    device does the same arithmetic: csrc/vm_device.cuh segment_of.)"""
    length, step = ray.length, cfg.segment_length
    if length <= step:
        return [ray]
    pieces = math.ceil(length / step)
    unit = (ray.end - ray.origin) / length
    starts = [ray.origin + unit * (i * step) for i in range(pieces)]
    ends = [ray.origin + unit * min((i + 1) * step, length) for i in range(pieces - 1)]
    ends.append(ray.end)
    flags = [False] * (pieces - 1) + [ray.has_sample]
    return [replace(ray, origin=o, end=e, has_sample=h) for o, e, h in zip(starts, ends, flags)]

"""NDT voxel Gaussian queries (mirror of voxmap.ndt queries, ndt.py:108-165).

The per-sample updates (Welford mean + Givens sqrt-covariance, miss
likelihood) run on the device: csrc/vm_kernels.cuh update_gaussian /
gaussian_weight.
"""
from __future__ import annotations

import numpy as np

from .keys import VoxelKey, voxel_min_corner
from .subvoxel import unpack_mean

MIN_SAMPLES_FOR_GAUSSIAN = 3


def sqrt_to_matrix(flat6) -> np.ndarray:
    s = np.asarray(flat6, dtype=np.float64)
    L = np.zeros((3, 3))
    L[0, 0] = s[0]
    L[1, 0], L[1, 1] = s[1], s[2]
    L[2, 0], L[2, 1], L[2, 2] = s[3], s[4], s[5]
    return L


def intensity_stats(n: int, mean: float, m2: float):
    if n == 0:
        return None
    return mean, m2 / n


def permeability(hits: int, misses: int) -> float | None:
    total = hits + misses
    return None if total == 0 else hits / total


def voxel_gaussian(vmap, key: VoxelKey):
    n = vmap.voxel_values("mean_count", key)
    if n is None or n == 0:
        return None
    cfg = vmap.cfg
    mu = voxel_min_corner(key, cfg) + unpack_mean(int(vmap.voxel_values("mean", key))) * cfg.voxel_size
    S = sqrt_to_matrix(vmap.voxel_values("cov_sqrt", key))
    return int(n), mu, S @ S.T


def voxel_permeability(vmap, key: VoxelKey) -> float | None:
    h = vmap.voxel_values("hit_count", key)
    m = vmap.voxel_values("miss_count", key)
    if h is None or m is None:
        return None
    return permeability(int(h), int(m))


def voxel_intensity_stats(vmap, key: VoxelKey):
    n = vmap.voxel_values("mean_count", key)
    vals = vmap.voxel_values("intensity", key)
    if n is None or vals is None:
        return None
    return intensity_stats(int(n), float(vals[0]), float(vals[1]))

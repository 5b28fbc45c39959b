"""NDT voxel Gaussians: queries (voxmap.ndt, ndt.py:108-165) and the host
mirror of the per-sample update.

The batch path updates Gaussians on the device (csrc/vm_ndt.cuh ndt_update:
Welford mean + Givens sqrt-covariance with CPython's hypot, per sample in ray
order; csrc/vm_kernels.cuh gaussian_weight for the miss likelihood).
`update_gaussian` is the same arithmetic on the host, for callers that fold
samples themselves.
"""
from __future__ import annotations

import math

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


def update_gaussian(n: int, mu, S, sample):
    """Fold one sample into (count, mean, sqrt-covariance) -- ndt.py:55-70.
    The deviation factor L = S * sqrt(n) takes the rank-one Welford term
    sqrt(n / (n + 1)) * (x - mu) by Givens rotations (cholupdate3,
    ndt.py:37-52), column by column; the population factor is L / sqrt(n + 1).
    With fewer than two samples the factor is zero."""
    x = np.asarray(sample, dtype=np.float64)
    if n == 0:
        return 1, x.copy(), np.zeros((3, 3))
    m = n + 1
    d = x - mu
    L = np.array(S, dtype=np.float64) * math.sqrt(n)
    v = d * math.sqrt(n / m)
    for k in range(3):
        r = math.hypot(L[k, k], v[k])
        if r == 0.0:
            continue
        c, s = L[k, k] / r, v[k] / r
        L[k, k] = r
        col, tail = L[k + 1:, k].copy(), v[k + 1:].copy()
        L[k + 1:, k] = c * col + s * tail
        v[k + 1:] = c * tail - s * col
    return m, mu + d / m, L / math.sqrt(m)


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

"""Shared helpers for the parity tests."""
from __future__ import annotations

import ast
import math
import hashlib
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load_cases():
    z = np.load(GOLDEN / "scenes.npz", allow_pickle=False)
    cases = []
    for i in range(int(z["ncases"])):
        p = f"c{i}_"
        nb = int(z[p + "nbatches"])
        digests = {k[len(p) + 7:]: str(z[k]) for k in z.files if k.startswith(p + "digest_")}
        cases.append(dict(name=str(z[p + "name"]), mode=str(z[p + "mode"]),
                          cfg=ast.literal_eval(str(z[p + "cfg"])),
                          batches=[z[p + f"b{j}"] for j in range(nb)], stats=z[p + "stats"],
                          regions=z[p + "regions"], digests=digests))
    return cases


def digest(region_keys, get_buf):
    """sha256 over sorted (region key, layer bytes) -- make_golden.layer_digest."""
    h = hashlib.sha256()
    for rk in sorted(region_keys):
        h.update(np.asarray(rk, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(get_buf(rk)).tobytes())
    return h.hexdigest()


def max_abs_diff(keys, get_a, get_b):
    worst, count = 0.0, 0
    for rk in keys:
        a = get_a(rk).astype(np.float64)
        b = get_b(rk).astype(np.float64)
        d = np.abs(a - b)
        if d.size:
            worst = max(worst, float(d.max()))
            count += int(np.count_nonzero(d))
    return worst, count


def hit_delta(cfg) -> float:
    """occupancy.hit_delta (occupancy.py:30-35): log-odds of p_hit."""
    return math.log(cfg.p_hit / (1.0 - cfg.p_hit))


def miss_delta(cfg) -> float:
    return math.log(cfg.p_miss / (1.0 - cfg.p_miss))


def clamp_fold(l0, k, delta, cmin, cmax):
    """k clamped f32 log-odds adds of `delta` per voxel (reference.py:22-23),
    vectorised; a voxel stops at its fixed point (the clamp)."""
    l = np.asarray(l0, dtype=np.float32).copy()
    k = np.asarray(k, dtype=np.int64)
    d, lo, hi = np.float32(delta), np.float32(cmin), np.float32(cmax)
    left = k.copy()
    idx = np.nonzero(left > 0)[0]
    while idx.size:
        old = l[idx]
        new = np.clip(old + d, lo, hi).astype(np.float32)
        l[idx] = new
        left[idx] -= 1
        keep = (left[idx] > 0) & (new != old)
        idx = idx[keep]
    return l


def cas_envelope(l0, hits, misses, cfg):
    """Bounds of any interleaving of `hits` hit updates and `misses` miss
    updates of one batch on each voxel: clamped adds are monotone, so all
    hits first then all misses gives the lowest result, all misses first the
    highest (swapping an adjacent (hit, miss) pair never lowers the result)."""
    h32, m32 = np.float32(hit_delta(cfg)), np.float32(miss_delta(cfg))
    lo = clamp_fold(clamp_fold(l0, hits, h32, cfg.clamp_min, cfg.clamp_max), misses, m32,
                    cfg.clamp_min, cfg.clamp_max)
    hi = clamp_fold(clamp_fold(l0, misses, m32, cfg.clamp_min, cfg.clamp_max), hits, h32,
                    cfg.clamp_min, cfg.clamp_max)
    # without clamping the two orders differ only by f32 rounding, either way
    return np.minimum(lo, hi), np.maximum(lo, hi)


# Reordering an unclamped run of f32 adds moves the result by rounding only:
# at most half an ulp of the largest intermediate (|l| <= 4) per add, in
# practice a few ulps of 4.0.  The slack is absolute.
ENVELOPE_SLACK = 8 * float(np.spacing(np.float32(4.0)))  # 3.8e-6 log-odds


def within_envelope(x, lo, hi, slack=ENVELOPE_SLACK):
    """Mask of x inside [lo - slack, hi + slack]."""
    x = np.asarray(x, dtype=np.float64)
    return (x >= np.asarray(lo, np.float64) - slack) & (x <= np.asarray(hi, np.float64) + slack)

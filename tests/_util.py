"""Shared helpers for the parity tests."""
from __future__ import annotations

import ast
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

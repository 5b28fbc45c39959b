"""CPU reference arm: the reference's own native kernel, driven like its engine.

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py cpu_baseline and
`bench.py --impl reference`).  Loads oracle/_ref/_kernels*.so -- the
reference's `voxmap._kernels` compiled unmodified from
/root/reference/pkg/src/voxmap/_kernels.pyx by oracle/build_ref.py -- and
calls `integrate_occupancy` (_kernels.pyx:376-470) exactly as
engine._run_parallel does (engine.py:240-262): contiguous chunks of
4 x workers segments on a ThreadPoolExecutor, region table from
engine._build_region_table's format (engine.py:121-147).

Preprocessing (clip + segment, engine.py:82-96) and region prefetch
(engine.py:99-118) are computed by the C port (oracle/vm_oracle.c) and are
NOT timed: the timed figure is the reference kernel alone, the strongest
CPU number (SURVEY.md section 8(d) "kernel-only").  When the compiled
reference kernel is unavailable the C port's sequential integrator is
timed instead (kind "port").
"""
from __future__ import annotations

import math
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

from . import oracle as orc
from .build_ref import built_path

REF_DIR = Path(__file__).resolve().parent / "_ref"


def load_ref_kernels():
    p = built_path()
    if p is None:
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import _kernels  # noqa: E402  (the reference's compiled module)
    return _kernels


def _pack(r):
    B, M = 1 << 20, (1 << 21) - 1
    return ((r[0] + B) & M) << 42 | ((r[1] + B) & M) << 21 | ((r[2] + B) & M)


class RefOccupancyRunner:
    """Reference native occupancy integration over a persistent region store."""

    def __init__(self, cfg, workers: int):
        self.k = load_ref_kernels()
        self.kind = "reference" if self.k is not None else "port"
        self.cfg = cfg
        self.workers = max(1, workers)
        self.vpr = cfg.region_dim ** 3
        self.regions = {}  # coord -> (occ, mean, count) numpy buffers
        self.oracle = None if self.k is not None else orc.OracleMap(cfg)
        self.pool = ThreadPoolExecutor(max_workers=self.workers)

    def close(self):
        self.pool.shutdown()

    def prepare(self, records):
        """Untimed: clip/segment + prefetch with the C port; region table."""
        o = records["origin"].astype(np.float64)
        e = records["end"].astype(np.float64)
        h = (records["flags"] & 1).astype(np.uint8)
        if self.k is None:
            return (o, e, h, records["intensity"].astype(np.float32))
        so, se, sh, _, processed = orc.preprocess(o, e, h, segment=True, cfg=self.cfg)
        for rc in orc.prefetch_regions(so, se, sh, cfg=self.cfg):
            key = tuple(int(c) for c in rc)
            if key not in self.regions:
                self.regions[key] = (np.zeros(self.vpr, np.float32), np.zeros(self.vpr, np.uint32),
                                     np.zeros(self.vpr, np.uint32))
        keys = sorted(self.regions)
        size = 8
        while size < 2 * max(len(keys), 1):
            size <<= 1
        tkeys = np.full(size, -1, np.int64)
        tvals = np.full(size, -1, np.int32)
        for idx, rk in enumerate(keys):
            key = _pack(rk)
            hh = self.k.hash_mix(key) & (size - 1)
            while tkeys[hh] != -1:
                hh = (hh + 1) & (size - 1)
            tkeys[hh] = key
            tvals[hh] = idx
        ptrs = [np.array([self.regions[rk][j].ctypes.data for rk in keys], dtype=np.intp)
                for j in range(3)]
        max_len = float(np.max(np.linalg.norm(se - so, axis=1))) if len(so) else 0.0
        cap = 3 * (int(math.ceil(max_len / self.cfg.voxel_size)) + 2) + 8
        return (so, se, sh, tkeys, tvals, ptrs, cap, processed)

    def run(self, prep):
        """Timed: the reference kernel over the prepared batch; returns
        (rays_processed, visits)."""
        if self.k is None:
            o, e, h, it = prep
            st = self.oracle.integrate(o, e, h, it, "occupancy")
            return st["rays_processed"], st["voxel_visits"]
        so, se, sh, tkeys, tvals, ptrs, cap, processed = prep
        n = len(so)
        chunks = self.workers * 4
        edges = np.linspace(0, n, chunks + 1).astype(int)
        empty = np.empty(0, dtype=np.intp)
        hit = math.log(self.cfg.p_hit / (1 - self.cfg.p_hit))
        miss = math.log(self.cfg.p_miss / (1 - self.cfg.p_miss))

        def task(a, b):
            return self.k.integrate_occupancy(
                so[a:b], se[a:b], sh[a:b], tkeys, tvals, ptrs[0], ptrs[1], ptrs[2], empty, empty,
                self.cfg.voxel_size, self.cfg.region_dim, hit, miss, self.cfg.clamp_min,
                self.cfg.clamp_max, 20, cap)

        futs = [self.pool.submit(task, int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])
                if b > a]
        visits = sum(f.result()[3] for f in futs)
        return processed, visits


def time_reference(cfg, batches, workers: int, budget_s: float = 20.0):
    """Time the reference kernel over as many batches as fit the budget.
    Returns dict(rays, visits, seconds, batches, kind, workers)."""
    runner = RefOccupancyRunner(cfg, workers)
    rays = visits = 0
    secs = 0.0
    used = 0
    try:
        for rec in batches:
            prep = runner.prepare(rec)
            t0 = time.perf_counter()
            r, v = runner.run(prep)
            secs += time.perf_counter() - t0
            rays += r
            visits += v
            used += 1
            if secs >= budget_s:
                break
    finally:
        runner.close()
    return dict(rays=rays, visits=visits, seconds=secs, batches=used, kind=runner.kind,
                workers=workers)

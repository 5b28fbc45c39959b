"""Synthetic lidar workloads of BASELINE.json's configs.

Deterministic per seed, numpy-vectorised, emitted as OHMB1 records
(rayset.RAY_DTYPE) exactly like a recorded ray set.  Geometry is shifted by
W0 = (204.8, 204.8, 204.8) m so no coordinate lands in region -1.

* C1 `os64_room_scan`: one Ouster-64 scan (64 x 2048 = 131,072 rays), sensor
  1.8 m above ground inside an open 30 x 24 m room with 6 m walls; 0.1 m.
* C2 `os128_canyon_batches`: Ouster-128 in a street canyon (facades at
  +-6 m, 15 m high, poles every 10 m), sensor moving 1 m/s along +x;
  1000 batches x 26,240 rays (128 beams x 205 columns = 10 ms of a 10 Hz
  rotation at 2.6 M rays/s); 0.05 m.
* C3 `os64_tunnel_scans`: Ouster-64 scans in a 4 x 3 m tunnel with 2 cm
  wall roughness, 0.5 m per scan; NDT-OM at 0.1 m.

Beam model: elevations linspace(-22.5, 22.5) deg, 2048 azimuth columns per
rotation, range noise N(0, 2 cm), intensity U(5, 50).  Returns up to 40 m
are kept at their true range (the reference clips >20 m to miss-only rays);
beams that hit nothing within 40 m are emitted at 40 m without a sample.
"""
from __future__ import annotations

import numpy as np

from .rayset import records_from_arrays

W0 = np.array([204.8, 204.8, 204.8])
MAX_RETURN = 40.0
COLUMNS = 2048


def _beam_dirs(beams: int, cols: np.ndarray, elev_deg=(-22.5, 22.5)):
    el = np.deg2rad(np.linspace(elev_deg[0], elev_deg[1], beams))
    az = 2.0 * np.pi * cols / COLUMNS
    el_g, az_g = np.meshgrid(el, az)  # column-major scan order: all beams of a column
    el_g, az_g = el_g.ravel(), az_g.ravel()
    return np.stack([np.cos(el_g) * np.cos(az_g), np.cos(el_g) * np.sin(az_g), np.sin(el_g)], 1)


def _plane_hit(o, d, axis, value, lo=None, hi=None):
    """t of the ray hitting plane x[axis] = value within the rectangle bounds."""
    with np.errstate(divide="ignore", invalid="ignore"):
        t = (value - o[:, axis]) / d[:, axis]
    t = np.where(t > 1e-9, t, np.inf)
    if lo is not None:
        p = o + d * np.where(np.isfinite(t), t, 0.0)[:, None]
        ok = np.all((p >= lo) & (p <= hi), axis=1)
        t = np.where(ok, t, np.inf)
    return t


def _cylinder_hit(o, d, cx, cy, r, h):
    fx, fy = o[:, 0] - cx, o[:, 1] - cy
    a = d[:, 0] ** 2 + d[:, 1] ** 2
    b = 2.0 * (fx * d[:, 0] + fy * d[:, 1])
    c = fx * fx + fy * fy - r * r
    disc = b * b - 4.0 * a * c
    with np.errstate(invalid="ignore", divide="ignore"):
        t = (-b - np.sqrt(disc)) / (2.0 * a)
    z = o[:, 2] + d[:, 2] * t
    ok = (disc >= 0) & (t > 1e-9) & (z >= 0.0) & (z <= h)
    return np.where(ok, t, np.inf)


def _emit(origins, d, t, rng, timestamps):
    n = len(d)
    hit = np.isfinite(t) & (t <= MAX_RETURN)
    rng_t = np.where(hit, t + rng.normal(0.0, 0.02, n), MAX_RETURN)
    rng_t = np.maximum(rng_t, 0.05)
    ends = origins + d * rng_t[:, None]
    return records_from_arrays(timestamps, origins + W0, ends + W0,
                               rng.uniform(5.0, 50.0, n).astype(np.float32), hit)


def os64_room_scan(seed: int = 0) -> np.ndarray:
    """C1: one OS1-64 scan, 131,072 rays (0.1 m voxels)."""
    rng = np.random.default_rng(seed)
    d = _beam_dirs(64, np.arange(COLUMNS))
    n = len(d)
    o = np.tile([0.0, 0.0, 1.8], (n, 1))
    t = _plane_hit(o, d, 2, 0.0)
    for axis, v in ((0, -15.0), (0, 15.0), (1, -12.0), (1, 12.0)):
        lo = np.array([-15.0, -12.0, 0.0])
        hi = np.array([15.0, 12.0, 6.0])
        t = np.minimum(t, _plane_hit(o, d, axis, v, lo - 1e-9, hi + 1e-9))
    return _emit(o, d, t, rng, np.arange(n) * 1e-7)


def _canyon_t(o, d):
    t = _plane_hit(o, d, 2, 0.0)
    for y in (-6.0, 6.0):
        t = np.minimum(t, _plane_hit(o, d, 1, y, np.array([-1e9, -7, 0.0]),
                                     np.array([1e9, 7, 15.0])))
    for px in np.arange(-20.0, 240.0, 10.0):
        for py in (-4.5, 4.5):
            t = np.minimum(t, _cylinder_hit(o, d, px, py, 0.1, 6.0))
    return t


def os128_canyon_batches(n_batches: int = 1000, cols_per_batch: int = 205, seed: int = 1,
                         speed: float = 1.0):
    """C2: list of record batches (128 beams x cols_per_batch columns each)."""
    rng = np.random.default_rng(seed)
    out = []
    for b in range(n_batches):
        cols = (b * cols_per_batch + np.arange(cols_per_batch)) % COLUMNS
        d = _beam_dirs(128, cols)
        t0 = b * 0.01
        x = speed * t0
        o = np.tile([x, 0.0, 1.8], (len(d), 1))
        out.append(_emit(o, d, _canyon_t(o, d), rng, t0 + np.arange(len(d)) * 3.8e-7))
    return out


BATCH_PERIOD = 0.1  # the reference CLI's batch period (cli.py:31)


def batch_by_period(records: np.ndarray, period: float = BATCH_PERIOD) -> list[np.ndarray]:
    """Cut a timestamp-ordered record stream into `period`-second batches, as
    the reference CLI's _load_batches does (cli.py:70-94)."""
    if len(records) == 0:
        return []
    ts = records["timestamp"]
    t0 = ts[0]
    edges = np.searchsorted(ts, t0 + period * np.arange(
        1, int(np.ceil((ts[-1] - t0) / period)) + 2))
    out, start = [], 0
    for edge in edges:
        if edge > start:
            out.append(records[start:edge])
            start = edge
        if start >= len(records):
            break
    return out


def os64_tunnel_scans(n_scans: int, seed: int = 2, step: float = 0.5):
    """C3: OS1-64 scans along a 4 x 3 m tunnel with rough walls."""
    rng = np.random.default_rng(seed)
    out = []
    d0 = _beam_dirs(64, np.arange(COLUMNS))
    for s in range(n_scans):
        o = np.tile([s * step, 0.0, 1.5], (len(d0), 1))
        t = np.full(len(d0), np.inf)
        lo = np.array([-1e9, -2.0, 0.0])
        hi = np.array([1e9, 2.0, 3.0])
        for axis, v in ((1, -2.0), (1, 2.0), (2, 0.0), (2, 3.0)):
            t = np.minimum(t, _plane_hit(o, d0, axis, v, lo - 1e-9, hi + 1e-9))
        t = t + rng.normal(0.0, 0.02, len(t))  # wall roughness
        out.append(_emit(o, d0, t, rng, s * 0.1 + np.arange(len(d0)) * 7.6e-7))
    return out


# ---------------------------------------------------------------- C4: UAV

def _heightfield(x, y):
    return 1.5 * np.sin(0.15 * x) * np.cos(0.1 * y) + 0.5 * np.sin(0.5 * x + 0.3 * y)


def _march_heightfield(o, d, t_max=MAX_RETURN, dt=0.25):
    """First t where the ray drops below the heightfield (vectorised march,
    then 40 bisection steps); inf when it never does within t_max."""
    n = len(d)
    t_hit = np.full(n, np.inf)
    prev = np.zeros(n)
    alive = np.ones(n, dtype=bool)
    for t in np.arange(dt, t_max + dt, dt):
        p = o + d * t
        below = alive & (p[:, 2] < _heightfield(p[:, 0], p[:, 1]))
        if below.any():
            lo, hi = prev[below].copy(), np.full(int(below.sum()), t)
            oo, dd = o[below], d[below]
            for _ in range(40):
                mid = 0.5 * (lo + hi)
                q = oo + dd * mid[:, None]
                under = q[:, 2] < _heightfield(q[:, 0], q[:, 1])
                hi = np.where(under, mid, hi)
                lo = np.where(under, lo, mid)
            t_hit[below] = hi
            alive &= ~below
        prev[:] = t
        if not alive.any():
            break
    return t_hit


def _tree_hit(o, d, trees):
    t = np.full(len(d), np.inf)
    for cx, cy, r, h in trees:
        base = float(_heightfield(np.float64(cx), np.float64(cy)))
        fx, fy = o[:, 0] - cx, o[:, 1] - cy
        a = d[:, 0] ** 2 + d[:, 1] ** 2
        b = 2.0 * (fx * d[:, 0] + fy * d[:, 1])
        c = fx * fx + fy * fy - r * r
        disc = b * b - 4.0 * a * c
        with np.errstate(invalid="ignore", divide="ignore"):
            tc = (-b - np.sqrt(disc)) / (2.0 * a)
        z = o[:, 2] + d[:, 2] * tc
        ok = (disc >= 0) & (tc > 1e-9) & (z >= base) & (z <= base + h)
        t = np.minimum(t, np.where(ok, tc, np.inf))
    return t


def uav_lawnmower_scans(n_scans: int, seed: int = 3, altitude: float = 10.0,
                        speed: float = 5.0, leg: float = 100.0, spacing: float = 20.0):
    """C4: OS1-64 scans from a UAV 10 m above a sinusoidal heightfield with
    trees, flying a lawnmower pattern (legs of `leg` m along x, `spacing` m
    apart); the sensor is pitched down 90 degrees, so its rotation sweeps the
    vertical plane across the track (upward beams return nothing)."""
    rng = np.random.default_rng(seed)
    tree_rng = np.random.default_rng(seed + 1000)
    nt = 400
    trees = np.stack([tree_rng.uniform(-20, leg + 20, nt), tree_rng.uniform(-20, 200, nt),
                      tree_rng.uniform(0.3, 1.0, nt), tree_rng.uniform(4.0, 9.0, nt)], 1)
    d0 = _beam_dirs(64, np.arange(COLUMNS))
    d0 = np.stack([d0[:, 2], d0[:, 1], -d0[:, 0]], 1)  # pitch down 90 deg about y
    out = []
    for s in range(n_scans):
        dist = s * speed * 0.1
        k = int(dist // leg)
        along = dist - k * leg
        x = along if k % 2 == 0 else leg - along
        y = k * spacing
        o = np.tile([x, y, float(_heightfield(np.float64(x), np.float64(y))) + altitude],
                    (len(d0), 1))
        near = trees[(np.abs(trees[:, 0] - x) < 45.0) & (np.abs(trees[:, 1] - y) < 45.0)]
        t = np.minimum(_march_heightfield(o, d0), _tree_hit(o, d0, near))
        out.append(_emit(o, d0, t, rng, s * 0.1 + np.arange(len(d0)) * 7.6e-7))
    return out


# ---------------------------------------------------------------- C5: town

TOWN_LOOP = (1200.0, 700.0)  # the driven rectangle (3.8 km perimeter)


def _town_buildings(seed: int):
    """Box buildings on a 40 m block grid with 12 m streets, the loop's
    streets kept clear: rows of (x0, y0, x1, y1, height)."""
    rng = np.random.default_rng(seed + 2000)
    out = []
    W, H = TOWN_LOOP
    for bx in np.arange(-200.0, W + 200.0, 40.0):
        for by in np.arange(-200.0, H + 200.0, 40.0):
            x0, y0 = bx + 6.0, by + 6.0
            x1, y1 = bx + 34.0, by + 34.0
            # keep the loop's corridors (|y| < 10 or |y - H| < 10 along x, same for x) open
            if min(abs(y0), abs(y1), abs(y0 - H), abs(y1 - H)) < 10.0 or \
               (y0 < 10.0 and y1 > -10.0) or (y0 < H + 10.0 and y1 > H - 10.0):
                continue
            if (x0 < 10.0 and x1 > -10.0) or (x0 < W + 10.0 and x1 > W - 10.0):
                continue
            if rng.uniform() < 0.15:
                continue  # an open lot
            out.append((x0, y0, x1, y1, rng.uniform(6.0, 20.0)))
    return np.array(out)


def _box_hit(o, d, box):
    x0, y0, x1, y1, h = box
    lo = np.array([x0, y0, 0.0])
    hi = np.array([x1, y1, h])
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        ta = (lo - o) * inv
        tb = (hi - o) * inv
    tmin = np.nanmax(np.minimum(ta, tb), axis=1)
    tmax = np.nanmin(np.maximum(ta, tb), axis=1)
    ok = (tmax >= tmin) & (tmin > 1e-9)
    return np.where(ok, tmin, np.inf)


def town_loop_position(s: int, step: float = 0.5):
    W, H = TOWN_LOOP
    p = (s * step) % (2 * (W + H))
    if p < W:
        return p, 0.0
    if p < W + H:
        return W, p - W
    if p < 2 * W + H:
        return W - (p - W - H), H
    return 0.0, H - (p - 2 * W - H)


def town_scans(first: int, n_scans: int, seed: int = 4, step: float = 0.5):
    """C5: OS1-64 scans `first` .. `first + n_scans - 1` of the 7,630-scan
    drive around a 3.8 km loop through a procedural town (ground, box
    buildings, tree cylinders), 0.5 m per scan.  Scan s is generated from
    its own seed, so any slice of the sequence is reproducible on its own."""
    blds = _town_buildings(seed)
    tree_rng = np.random.default_rng(seed + 3000)
    W, H = TOWN_LOOP
    nt = 1500
    side = tree_rng.integers(0, 4, nt)
    u = tree_rng.uniform(0, 1, nt)
    off = tree_rng.choice([-7.0, 7.0], nt)
    tx = np.where(side == 0, u * W, np.where(side == 1, W + off, np.where(side == 2, u * W, off)))
    ty = np.where(side == 0, off, np.where(side == 1, u * H, np.where(side == 2, H + off, u * H)))
    trees = np.stack([tx, ty, tree_rng.uniform(0.2, 0.5, nt), tree_rng.uniform(4.0, 8.0, nt)], 1)
    d0 = _beam_dirs(64, np.arange(COLUMNS))
    out = []
    for s in range(first, first + n_scans):
        rng = np.random.default_rng([seed, s])
        x, y = town_loop_position(s, step)
        o = np.tile([x, y, 1.8], (len(d0), 1))
        t = _plane_hit(o, d0, 2, 0.0)
        near = blds[(np.abs(0.5 * (blds[:, 0] + blds[:, 2]) - x) < 65.0) &
                    (np.abs(0.5 * (blds[:, 1] + blds[:, 3]) - y) < 65.0)]
        for b in near:
            t = np.minimum(t, _box_hit(o, d0, b))
        nt_ = trees[(np.abs(trees[:, 0] - x) < 45.0) & (np.abs(trees[:, 1] - y) < 45.0)]
        for cx, cy, r, h in nt_:
            t = np.minimum(t, _cylinder_hit(o, d0, cx, cy, r, h))
        out.append(_emit(o, d0, t, rng, s * 0.1 + np.arange(len(d0)) * 7.6e-7))
    return out


TOWN_SCANS = 7630  # x 131,072 rays = 1,000,079,360 (BASELINE configs[4])
UAV_SCANS = 382    # x 131,072 rays = 50,069,504 (configs[3])

"""The BASELINE workload generators (paper_2206_06079_b200/scans.py) on CPU:
deterministic per seed, the configs' sizes, and geometry that produces the
evidence each config is about (samples, clipped miss-only rays, W0 offset)."""
import numpy as np

from paper_2206_06079_b200 import scans
from paper_2206_06079_b200.rayset import RAY_DTYPE


def _check(rec, n=131072):
    assert rec.dtype == RAY_DTYPE and len(rec) == n
    o = rec["origin"].astype(np.float64)
    e = rec["end"].astype(np.float64)
    L = np.linalg.norm(e - o, axis=1)
    assert np.all(L > 0) and np.all(L <= scans.MAX_RETURN + 0.5)
    assert np.all(e > 100.0)  # shifted by W0: no coordinate in region -1
    has = (rec["flags"] & 1) == 1
    return has, L


def test_c1_c3_generators_deterministic():
    a, b = scans.os64_room_scan(seed=0), scans.os64_room_scan(seed=0)
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    has, L = _check(a)
    assert 0.8 < has.mean() < 0.9  # 85% returns
    t = scans.os64_tunnel_scans(2)
    has, _ = _check(t[1])
    assert has.mean() > 0.9


def test_c4_uav_lawnmower():
    s = scans.uav_lawnmower_scans(2)
    again = scans.uav_lawnmower_scans(2)
    assert np.array_equal(s[1].view(np.uint8), again[1].view(np.uint8))
    has, L = _check(s[0])
    # pitched-down sensor: the lower half of the sweep returns from the
    # terrain / trees, the upper half sees sky (40 m miss-only rays)
    assert 0.35 < has.mean() < 0.6
    assert np.any(L > 20.0)
    assert scans.UAV_SCANS * 131072 >= 50_000_000
    # the UAV moves 0.5 m per scan along the lawnmower leg
    assert abs(float(s[1]["origin"][0, 0] - s[0]["origin"][0, 0]) - 0.5) < 1e-4


def test_c5_town_loop():
    a = scans.town_scans(0, 2)
    b = scans.town_scans(1, 1)  # a slice of the sequence regenerates on its own
    assert np.array_equal(a[1].view(np.uint8), b[0].view(np.uint8))
    has, _ = _check(a[0])
    assert 0.4 < has.mean() < 0.95
    assert scans.TOWN_SCANS * 131072 == 1_000_079_360
    W, H = scans.TOWN_LOOP
    assert abs(2 * (W + H) - 3800.0) < 1e-9
    # the drive closes the loop
    assert scans.town_loop_position(0) == scans.town_loop_position(int(3800 / 0.5))

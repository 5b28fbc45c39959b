"""CPU check of the order envelope the CAS parity tests rely on
(tests/test_gpu_cas.py): every interleaving of a voxel's hits and misses,
folded with the reference's clamped f32 update (reference.py:22-23), lies
between "all hits first" and "all misses first"."""
import numpy as np

from paper_2206_06079_b200 import MapConfig
from tests._util import cas_envelope, clamp_fold, hit_delta, miss_delta, within_envelope


def _seq_fold(l, seq, cfg):
    h32, m32 = np.float32(hit_delta(cfg)), np.float32(miss_delta(cfg))
    lo, hi = np.float32(cfg.clamp_min), np.float32(cfg.clamp_max)
    l = np.float32(l)
    for is_hit in seq:
        l = np.float32(min(max(np.float32(l + (h32 if is_hit else m32)), lo), hi))
    return l


def test_clamp_fold_matches_sequential():
    cfg = MapConfig()
    rng = np.random.default_rng(3)
    l0 = rng.uniform(-2, 3.5, 500).astype(np.float32)
    k = rng.integers(0, 40, 500)
    got = clamp_fold(l0, k, miss_delta(cfg), cfg.clamp_min, cfg.clamp_max)
    for i in range(500):
        assert got[i] == _seq_fold(l0[i], [False] * int(k[i]), cfg)


def test_every_interleaving_inside_envelope():
    cfg = MapConfig()
    rng = np.random.default_rng(11)
    n = 3000
    l0 = rng.uniform(-2, 3.5, n).astype(np.float32)
    l0[:200] = np.float32(cfg.clamp_min)
    l0[200:400] = np.float32(cfg.clamp_max)
    hits = rng.integers(0, 7, n)
    misses = rng.integers(0, 25, n)
    lo, hi = cas_envelope(l0, hits, misses, cfg)
    assert np.all(lo <= hi)
    got = np.empty(n, dtype=np.float32)
    for i in range(n):
        seq = np.array([True] * int(hits[i]) + [False] * int(misses[i]))
        rng.shuffle(seq)
        got[i] = _seq_fold(l0[i], seq, cfg)
    assert within_envelope(got, lo, hi).all()
    # single-kind voxels are order-free: the envelope collapses to a point
    single = (hits == 0) | (misses == 0)
    assert np.array_equal(lo[single], hi[single])
    assert (hi - lo > 1e-3).sum() > 100  # the envelope is not vacuous: clamping bites
    assert np.array_equal(got[single], lo[single])

"""The C oracle (oracle/vm_oracle.c) against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests._util import digest, load_cases

from tests._util import GOLDEN

STAT_KEYS = ("rays_in", "rays_processed", "segments", "voxel_visits", "cas_retries",
             "cas_failures", "region_misses", "regions_touched")


def test_walk_vectors_bit_exact():
    z = np.load(GOLDEN / "walk.npz")
    pts, off = z["pts"], z["offsets"]
    for i, p in enumerate(pts):
        c, t0, t1 = orc.walk(p[:3], p[3:], float(z["cell"]))
        a, b = off[i], off[i + 1]
        assert np.array_equal(c, z["coords"][a:b]), i
        assert np.array_equal(t0.view(np.uint64), z["t0"][a:b].view(np.uint64)), i
        assert np.array_equal(t1.view(np.uint64), z["t1"][a:b].view(np.uint64)), i


def test_corner_tie_break_kat():
    # test_kernels.py:25-27, test_traversal.py:30-42
    c, _, _ = orc.walk((0.05, 0.05, 0.05), (0.15, 0.15, 0.15), 0.1)
    assert c.tolist() == [[0, 0, 0], [1, 0, 0], [1, 1, 0], [1, 1, 1]]
    c, t0, t1 = orc.walk((0.05, 0.05, 0.05), (0.15, 0.15, 0.05), 0.1)
    assert c.tolist() == [[0, 0, 0], [1, 0, 0], [1, 1, 0]] and t1[1] == t0[1]


def test_norm_and_hypot_vectors():
    z = np.load(GOLDEN / "arith.npz")
    got = np.array([orc.norm3(*v) for v in z["v"]])
    assert np.array_equal(got.view(np.uint64), z["norms"].view(np.uint64))
    got = np.array([orc.py_hypot(a, b) for a, b in z["hy"]])
    assert np.array_equal(got.view(np.uint64), z["hyp"].view(np.uint64))


def test_clip_segment_vectors():
    z = np.load(GOLDEN / "arith.npz")
    rec = z["seg_records"]
    o = rec["origin"].astype(np.float64)
    e = rec["end"].astype(np.float64)
    h = (rec["flags"] & 1).astype(np.uint8)
    so, se, sh, sr, _ = orc.preprocess(o, e, h, segment=True)
    assert np.array_equal(so.view(np.uint64), z["seg_o"].view(np.uint64))
    assert np.array_equal(se.view(np.uint64), z["seg_e"].view(np.uint64))
    assert np.array_equal(sh, z["seg_has"]) and np.array_equal(sr, z["seg_ray"])
    # clipped rays that round above 20 m gain the degenerate third segment
    assert np.bincount(np.bincount(sr)).size >= 4


CASES = load_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_sequential_reference_golden(case):
    om = orc.OracleMap(None, orc.MODE_LAYERS[case["mode"]], **case["cfg"])
    for j, b in enumerate(case["batches"]):
        st = om.integrate_records(b, case["mode"])
        assert [st[k] for k in STAT_KEYS] == case["stats"][j].tolist()
    keys = om.region_keys()
    assert sorted(keys) == [tuple(r) for r in case["regions"].tolist()]
    for name, d in case["digests"].items():
        assert digest(keys, lambda rk: om.layer(rk, name)) == d, name

"""CAS-mode parity (the paper's lock-free clamped update, _kernels.pyx:233-357)
made falsifiable voxel by voxel.

Per batch, the C oracle counts every voxel's hit and miss visits (its
"counts" checker mode, the visits integrate_occupancy_segment makes).  From
the voxel's log-odds before the batch, any interleaving of those updates
lies between "all hits first" and "all misses first" (tests/_util.py
cas_envelope; tests/test_cas_envelope.py checks the claim on random
sequences).  So for every voxel:

* only misses, or only hits (order-free: identical deltas commute): the CAS
  result is bit-exact -- on the reference's mixed-free corridor this is the
  whole map (test_engine.py:52-55, SURVEY finding 4);
* both: the CAS result lies inside the envelope (plus a few f32 ulps of
  rounding).

mean_count is exact everywhere (a fetch-add per hit).
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests._util import cas_envelope, clamp_fold, load_cases, miss_delta, hit_delta, within_envelope

pytestmark = pytest.mark.gpu

from paper_2206_06079_b200 import ExecutorOptions, MapConfig, VoxelMap, scans, submit_batch  # noqa
from paper_2206_06079_b200.layers import MODE_LAYERS  # noqa: E402

OCC_CASES = [c for c in load_cases() if c["mode"] in ("occupancy", "decay")]


def _snapshot(vm):
    return {rk: r.buffers["occupancy"].copy() for rk, r in vm.regions.items()}


def _batch_counts(cfg, rec):
    om = orc.OracleMap(cfg, orc.MODE_LAYERS["counts"])
    om.integrate_records(rec, "counts")
    return {rk: (om.layer(rk, "hit_count"), om.layer(rk, "miss_count")) for rk in om.region_keys()}


def run_cas_with_envelope(cfg, batches, mode="occupancy"):
    """Integrate `batches` in CAS mode, checking each batch against its
    envelope; returns (map, mixed voxels, max envelope width seen, max
    distance from the sequential result)."""
    vm = VoxelMap(cfg, MODE_LAYERS[mode])
    om = orc.OracleMap(cfg, MODE_LAYERS[mode])
    vpr = cfg.region_dim ** 3
    mixed = 0
    for rec in batches:
        before = _snapshot(vm)
        st = submit_batch(vm, rec, mode, ExecutorOptions(deterministic=False))
        ost = om.integrate_records(rec, mode)
        assert st.voxel_visits == ost["voxel_visits"] and st.region_misses == 0
        assert st.cas_failures == 0
        counts = _batch_counts(cfg, rec)
        for rk, region in vm.regions.items():
            l1 = region.buffers["occupancy"]
            l0 = before.get(rk, np.zeros(vpr, np.float32))
            h, k = counts.get(rk, (np.zeros(vpr, np.uint32), np.zeros(vpr, np.uint32)))
            lo, hi = cas_envelope(l0, h, k, cfg)
            free = (h == 0) | (k == 0)
            # order-free voxels: bit-exact
            assert np.array_equal(l1[free].view(np.uint32), lo[free].view(np.uint32)), rk
            ok = within_envelope(l1, lo, hi)
            assert ok.all(), (rk, int((~ok).sum()))
            mixed += int(np.count_nonzero(~free))
    assert set(vm.regions) == set(om.region_keys())
    dev = 0.0
    for rk, region in vm.regions.items():
        assert np.array_equal(region.buffers["mean_count"], om.layer(rk, "mean_count")), rk
        if mode == "decay":
            assert np.array_equal(region.buffers["decay_hits"], om.layer(rk, "decay_hits")), rk
            d = np.abs(region.buffers["decay_distance"] - om.layer(rk, "decay_distance"))
            assert d.max(initial=0.0) <= 1e-9, rk
        d = np.abs(region.buffers["occupancy"].astype(np.float64) - om.layer(rk, "occupancy"))
        dev = max(dev, float(d.max(initial=0.0)))
    return vm, mixed, dev


@pytest.mark.parametrize("case", OCC_CASES, ids=[c["name"] for c in OCC_CASES])
def test_cas_golden_inside_order_envelope(case):
    cfg = MapConfig(**case["cfg"])
    _, mixed, dev = run_cas_with_envelope(cfg, case["batches"], case["mode"])
    if case["name"].startswith("corridor"):
        # the reference's mixed-free scene: CAS equals sequential bit for bit
        assert mixed == 0 and dev == 0.0


def test_clamp_fold_helper_matches_device_semantics():
    """f_miss^k of the checker equals the oracle's sequential fold."""
    cfg = MapConfig()
    rng = np.random.default_rng(1)
    l0 = rng.uniform(-2, 3.5, 64).astype(np.float32)
    k = rng.integers(0, 30, 64)
    got = clamp_fold(l0, k, miss_delta(cfg), cfg.clamp_min, cfg.clamp_max)
    ref = l0.copy()
    for i in range(64):
        for _ in range(int(k[i])):
            ref[i] = np.float32(min(max(np.float32(ref[i] + np.float32(miss_delta(cfg))),
                                        np.float32(cfg.clamp_min)), np.float32(cfg.clamp_max)))
    assert np.array_equal(got, ref)
    assert np.float32(hit_delta(cfg)) == np.float32(0.8472978603872037)


@pytest.mark.slow
def test_c2_prefix_cas_inside_order_envelope():
    """Three C2 batches at 0.05 m (787k rays, ~215 M visits): every voxel
    without both hits and misses is bit-exact, every mixed voxel inside its
    envelope."""
    cfg = MapConfig(voxel_size=0.05)
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(30)))[:3]
    _, mixed, dev = run_cas_with_envelope(cfg, data)
    assert mixed > 1000  # the canyon does mix hits and misses
    print(f"CAS C2 prefix: {mixed} mixed voxel-batches, max |CAS - sequential| {dev:.4f}")

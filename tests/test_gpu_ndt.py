"""NDT-OM / NDT-TM parity.

The device replays the reference's NDT phase 2 sample by sample -- Welford
mean plus the Givens rank-one update cholupdate3 with CPython's math.hypot
(ndt.py:37-70, reference.py:107-150) -- in ray order per voxel (vm_ndt.cuh).
Deterministic mode is therefore held to the reference's own golden layer
digests (every layer, mean and cov_sqrt included) and to the C oracle on
full tunnel scans, bit for bit.

CAS mode applies phase 1 with per-visit atomics, so misses through a
Gaussian voxel land in arbitrary order; phase 2 is the same ordered fold.
As in the reference's own test (test_engine.py:61-63: NDT mean and cov exact
across executors) mean, mean_count and cov_sqrt are exact; occupancy is
bounded by 1e-4 (test_engine.py:52-55).
"""
import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests._util import digest, load_cases

pytestmark = pytest.mark.gpu

from paper_2206_06079_b200 import ExecutorOptions, MapConfig, VoxelMap, scans, submit_batch  # noqa
from paper_2206_06079_b200.layers import MODE_LAYERS  # noqa: E402

NDT_CASES = [c for c in load_cases() if c["mode"].startswith("ndt")]


def _gpu(batches, cfg, mode, det):
    vm = VoxelMap(cfg, MODE_LAYERS[mode])
    stats = [submit_batch(vm, b, mode, ExecutorOptions(deterministic=det)) for b in batches]
    return vm, stats


def _oracle(batches, cfg, mode):
    om = orc.OracleMap(cfg, MODE_LAYERS[mode])
    stats = [om.integrate_records(b, mode) for b in batches]
    return om, stats


def _assert_layers_equal(vm, om, names, skip=()):
    assert set(vm.regions) == set(om.region_keys())
    for rk, region in vm.regions.items():
        for name in names:
            if name in skip:
                continue
            a, b = region.buffers[name], om.layer(rk, name)
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (rk, name)


@pytest.mark.parametrize("case", NDT_CASES, ids=[c["name"] for c in NDT_CASES])
def test_ndt_deterministic_bit_exact_to_reference_golden(case):
    """Every layer's digest equals the one the reference's sequential
    executor produced (tests/golden/make_golden.py)."""
    vm, stats = _gpu(case["batches"], MapConfig(**case["cfg"]), case["mode"], True)
    for j, st in enumerate(stats):
        want = case["stats"][j].tolist()
        got = [st.rays_in, st.rays_processed, st.segments, st.voxel_visits, want[4],
               st.cas_failures, st.region_misses, st.regions_touched]
        assert got == want, (j, got, want)
    keys = list(vm.regions)
    assert sorted(keys) == [tuple(r) for r in case["regions"].tolist()]
    for name, d in case["digests"].items():
        assert digest(keys, lambda rk: vm.regions[rk].buffers[name]) == d, name


@pytest.mark.parametrize("case", NDT_CASES, ids=[c["name"] for c in NDT_CASES])
def test_ndt_cas_mean_cov_exact(case):
    cfg = MapConfig(**case["cfg"])
    vm, stats = _gpu(case["batches"], cfg, case["mode"], False)
    om, ostats = _oracle(case["batches"], cfg, case["mode"])
    assert [s.voxel_visits for s in stats] == [s["voxel_visits"] for s in ostats]
    assert all(s.region_misses == 0 for s in stats)
    names = MODE_LAYERS[case["mode"]]
    _assert_layers_equal(vm, om, names, skip=("occupancy", "miss_count", "intensity"))
    for rk, region in vm.regions.items():
        d = np.abs(region.buffers["occupancy"].astype(np.float64) - om.layer(rk, "occupancy"))
        assert d.max(initial=0.0) <= 1e-4, rk
        if "miss_count" in names and case["name"].startswith("corridor"):
            # a transient reset zeroes the miss count mid-batch: with CAS the
            # count kept depends on which misses land after it
            assert np.array_equal(region.buffers["miss_count"], om.layer(rk, "miss_count")), rk
        if "intensity" in names:
            d = np.abs(region.buffers["intensity"].astype(np.float64) - om.layer(rk, "intensity"))
            assert d.max(initial=0.0) <= 1e-9, rk


@pytest.mark.slow
def test_c3_ten_tunnel_scans_bit_exact():
    """Ten C3 scans (1.31 M rays): Gaussians form on the rough walls from the
    second scan on, so phase-1 weights, resets and per-sample Givens
    updates with up to hundreds of samples per voxel are all exercised."""
    data = scans.os64_tunnel_scans(10)
    vm, stats = _gpu(data, MapConfig(), "ndt-om", True)
    om, ostats = _oracle(data, MapConfig(), "ndt-om")
    for s, o in zip(stats, ostats):
        assert (s.voxel_visits, s.segments, s.rays_processed) == \
            (o["voxel_visits"], o["segments"], o["rays_processed"])
        assert s.region_misses == 0
    assert sum(s.records for s in stats) > sum(s.rays_processed for s in stats[1:])  # phase-1 records
    _assert_layers_equal(vm, om, MODE_LAYERS["ndt-om"])


@pytest.mark.slow
def test_c1_ndt_tm_bit_exact():
    data = [scans.os64_room_scan(seed=0)[::2].copy(), scans.os64_room_scan(seed=5)[1::2].copy()]
    vm, _ = _gpu(data, MapConfig(), "ndt-tm", True)
    om, _ = _oracle(data, MapConfig(), "ndt-tm")
    _assert_layers_equal(vm, om, MODE_LAYERS["ndt-tm"])


@pytest.mark.slow
def test_ndt_record_overflow_replay(monkeypatch):
    """Records (and voxel indices) that overflow their buffers: the batch
    re-emits its records into grown buffers and folds them; nothing is
    applied twice (the replay must not re-count the ray-order
    histogram)."""
    data = scans.os64_tunnel_scans(3)
    ref, _ = _gpu(data, MapConfig(), "ndt-om", True)
    monkeypatch.setenv("VOXMAP_B200_TEST_NDT_REC_CAP", "4096")
    small, stats = _gpu(data, MapConfig(), "ndt-om", True)
    assert max(s.records for s in stats) > 4096
    assert set(ref.regions) == set(small.regions)
    for rk, region in ref.regions.items():
        for name in MODE_LAYERS["ndt-om"]:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  small.regions[rk].buffers[name].view(np.uint8)), (rk, name)
    # the next batch after a replay still walks every ray once
    more = scans.os64_tunnel_scans(4)[3:]
    s1 = submit_batch(ref, more[0], "ndt-om")
    s2 = submit_batch(small, more[0], "ndt-om")
    assert s1.voxel_visits == s2.voxel_visits and s1.records == s2.records
    assert os.environ.get("VOXMAP_B200_TEST_NDT_REC_CAP") == "4096"


NDT_STAT_FIELDS = ("rays_in", "rays_processed", "segments", "voxel_visits", "region_misses",
                   "regions_touched", "records", "marked_voxels", "new_regions")


def _sequence_vs_single(batches, mode, cfg, **kw):
    """submit_batches (one pipelined device sequence, vm_integrate_many) against
    one submit_batch per batch: the same stats and the same bits."""
    from paper_2206_06079_b200 import submit_batches
    a = VoxelMap(cfg, MODE_LAYERS[mode], **kw)
    b = VoxelMap(cfg, MODE_LAYERS[mode], **kw)
    sa = submit_batches(a, batches, mode)
    sb = [submit_batch(b, x, mode) for x in batches]
    for i, (x, y) in enumerate(zip(sa, sb)):
        gx = {k: getattr(x, k) for k in NDT_STAT_FIELDS}
        gy = {k: getattr(y, k) for k in NDT_STAT_FIELDS}
        assert gx == gy, (i, {k: (gx[k], gy[k]) for k in NDT_STAT_FIELDS if gx[k] != gy[k]})
    assert set(a.regions) == set(b.regions)
    for rk, region in a.regions.items():
        for name in MODE_LAYERS[mode]:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  b.regions[rk].buffers[name].view(np.uint8)), (rk, name)
    return sa, a


@pytest.mark.parametrize("mode", ["ndt-om", "ndt-tm"])
def test_ndt_pipelined_sequence_matches_per_batch(mode):
    """NDT sequences run as one pipelined device sequence; a tiny initial
    region pool forces mid-sequence refusals (grow + replay from that batch,
    its voxel-index claims kept) and an empty batch sits in the middle.
    (0.04 m voxels: 1.28 m regions, about a thousand per scan.)"""
    data = scans.os64_tunnel_scans(5)
    seq = [data[0], data[1][:0], data[1], data[2], data[3], data[4]]
    sa, _ = _sequence_vs_single(seq, mode, MapConfig(voxel_size=0.04), initial_regions=64)
    assert any(s.replays for s in sa)
    assert sum(s.records for s in sa) > 0


@pytest.mark.slow
def test_ndt_pipelined_sequence_record_overflow(monkeypatch):
    """Records / voxel indices overflowing mid-sequence stop the chain at that
    batch; it is re-emitted into grown buffers and folded, the rest
    re-enqueued -- the bits of an unconstrained per-batch run."""
    from paper_2206_06079_b200 import submit_batches
    data = scans.os64_tunnel_scans(4)
    ref = VoxelMap(MapConfig(), MODE_LAYERS["ndt-om"])
    want = [submit_batch(ref, x, "ndt-om") for x in data]
    monkeypatch.setenv("VOXMAP_B200_TEST_NDT_REC_CAP", "4096")
    vm = VoxelMap(MapConfig(), MODE_LAYERS["ndt-om"])
    got = submit_batches(vm, data, "ndt-om")
    assert max(s.records for s in got) > 4096
    for x, y in zip(got, want):
        assert (x.voxel_visits, x.records, x.marked_voxels) == (y.voxel_visits, y.records, y.marked_voxels)
    assert set(vm.regions) == set(ref.regions)
    for rk, region in ref.regions.items():
        for name in MODE_LAYERS["ndt-om"]:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  vm.regions[rk].buffers[name].view(np.uint8)), (rk, name)


@pytest.mark.slow
def test_ndt_pipelined_c3_against_oracle():
    """Eight C3 scans through submit_batches against the C oracle, bit for bit."""
    from paper_2206_06079_b200 import submit_batches
    data = scans.os64_tunnel_scans(8)
    vm = VoxelMap(MapConfig(), MODE_LAYERS["ndt-om"])
    stats = submit_batches(vm, data, "ndt-om")
    om, ostats = _oracle(data, MapConfig(), "ndt-om")
    for s, o in zip(stats, ostats):
        assert (s.voxel_visits, s.segments, s.rays_processed) == \
            (o["voxel_visits"], o["segments"], o["rays_processed"])
    _assert_layers_equal(vm, om, MODE_LAYERS["ndt-om"])

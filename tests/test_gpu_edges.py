"""GPU parity on edge cases and at full size: the deterministic path must be
bit-exact to the C oracle (a restatement of sequential_reference,
reference.py:35-64 / engine.py:222-237) on

* hot sample voxels -- thousands of rays ending in one voxel while others
  pass through it -- which exercise the three fold paths of vm_bucket.cuh
  (thread insertion sort <= 16 records, block bitonic sort <= 4096, order
  bitmaps above);
* empty, zero-length, miss-only, clipped (> max range) and single-ray batches
  (engine.py:82-96, traversal.py:140-178);
* a full C1 scan (131,072 rays, 25M visits) and a 3-batch C2 prefix at 0.05 m.
"""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

from paper_2206_06079_b200 import ExecutorOptions, MapConfig, VoxelMap, scans, submit_batch  # noqa
from paper_2206_06079_b200.layers import MODE_LAYERS  # noqa: E402
from paper_2206_06079_b200.rayset import records_from_arrays  # noqa: E402

W0 = np.array([204.8, 204.8, 204.8])


def _recs(o, e, has, inten=None):
    n = len(o)
    inten = np.full(n, 10.0) if inten is None else inten
    return records_from_arrays(np.zeros(n), o, e, inten, has)


def _compare(batches, cfg=None, mode="occupancy", det=True):
    cfg = cfg or MapConfig()
    names = MODE_LAYERS[mode]
    vm = VoxelMap(cfg, names)
    om = orc.OracleMap(cfg, names)
    for rec in batches:
        st = submit_batch(vm, rec, mode, ExecutorOptions(deterministic=det))
        ost = om.integrate_records(rec, mode)
        assert st.voxel_visits == ost["voxel_visits"]
        assert st.segments == ost["segments"]
        assert st.rays_processed == ost["rays_processed"]
        assert st.region_misses == 0
    assert set(vm.regions) == set(om.region_keys())
    for rk, region in vm.regions.items():
        for name in names:
            a, b = region.buffers[name], om.layer(rk, name)
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (rk, name)
    return vm


def _hot_voxel_batch(rng, n_hit, n_pass, target):
    """n_hit rays from random origins ending at `target`'s voxel, n_pass rays
    crossing it; ray order is shuffled so hits and misses interleave."""
    d = rng.normal(size=(n_hit, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o_hit = target + d * rng.uniform(2.0, 15.0, (n_hit, 1))
    e_hit = target + rng.uniform(-0.04, 0.04, (n_hit, 3))
    d2 = rng.normal(size=(n_pass, 3))
    d2 /= np.linalg.norm(d2, axis=1, keepdims=True)
    o_pass = target - d2 * rng.uniform(1.0, 8.0, (n_pass, 1))
    e_pass = target + d2 * rng.uniform(1.0, 8.0, (n_pass, 1))
    o = np.concatenate([o_hit, o_pass])
    e = np.concatenate([e_hit, e_pass])
    has = np.concatenate([np.ones(n_hit, bool), rng.random(n_pass) < 0.5])
    p = rng.permutation(len(o))
    return _recs(o[p], e[p], has[p])


@pytest.mark.parametrize("n_hit,n_pass", [(5, 8), (40, 300), (900, 2500), (3000, 9000)],
                         ids=["thread", "block-small", "block-large", "bitmap"])
def test_hot_sample_voxel_fold_paths(n_hit, n_pass):
    rng = np.random.default_rng(n_hit)
    target = W0 + np.array([3.05, 2.05, 1.05])
    batches = [_hot_voxel_batch(rng, n_hit, n_pass, target) for _ in range(2)]
    _compare(batches)


def test_many_hot_voxels_mixed_sizes():
    rng = np.random.default_rng(11)
    parts = []
    for k in range(24):
        t = W0 + rng.uniform(-6, 6, 3)
        parts.append(_hot_voxel_batch(rng, int(rng.integers(1, 600)), int(rng.integers(0, 2000)), t))
    rec = np.concatenate(parts)
    rec = rec[rng.permutation(len(rec))]
    _compare([rec, rec[::-1].copy()])


def test_degenerate_batches():
    rng = np.random.default_rng(3)
    o = W0 + rng.uniform(-1, 1, (64, 3))
    e = o + rng.normal(size=(64, 3)) * 5
    empty = _recs(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0, bool))
    zero_len = _recs(o, o.copy(), np.ones(64, bool))
    miss_only = _recs(o, e, np.zeros(64, bool))
    far = e + (e - o) * 6.0  # > 20 m: clipped, miss-only (traversal.py:140-150)
    clipped = _recs(o, far, np.ones(64, bool))
    single = _recs(o[:1], e[:1], np.ones(1, bool))
    exact = _recs(np.round(o * 10) / 10, np.round(e * 10) / 10, np.ones(64, bool))  # on faces
    _compare([empty, zero_len, miss_only, clipped, single, exact, empty])


def test_cas_degenerate_batches_order_free_layers():
    rng = np.random.default_rng(4)
    o = W0 + rng.uniform(-1, 1, (256, 3))
    e = o + rng.normal(size=(256, 3)) * 8
    vm = VoxelMap(MapConfig(), MODE_LAYERS["occupancy"])
    st = submit_batch(vm, _recs(o, e, np.zeros(256, bool)), "occupancy",
                      ExecutorOptions(deterministic=False))
    om = orc.OracleMap(MapConfig(), MODE_LAYERS["occupancy"])
    om.integrate_records(_recs(o, e, np.zeros(256, bool)))
    assert st.region_misses == 0
    for rk, region in vm.regions.items():  # miss-only: order-free, exact
        assert np.array_equal(region.buffers["occupancy"], om.layer(rk, "occupancy"))


@pytest.mark.slow
def test_full_c1_scan_bit_exact():
    _compare([scans.os64_room_scan(seed=0)])


@pytest.mark.slow
def test_c2_prefix_bit_exact():
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(30)))
    _compare(data[:3], cfg=MapConfig(voxel_size=0.05))


@pytest.mark.slow
def test_c2_twenty_batches_pipelined_bit_exact():
    """20 of C2's 100 batches (5.2 M rays, ~1.4 G visits, 2 s of sensor time)
    through the bench's own path -- submit_batches, one pipelined device
    sequence -- against the C oracle: region set and every layer bit-exact."""
    from paper_2206_06079_b200 import submit_batches
    cfg = MapConfig(voxel_size=0.05)
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(200)))[:20]
    assert len(data) == 20
    names = MODE_LAYERS["occupancy"]
    vm = VoxelMap(cfg, names, initial_regions=4096)
    om = orc.OracleMap(cfg, names)
    sts = submit_batches(vm, data, "occupancy")
    for st, rec in zip(sts, data):
        ost = om.integrate_records(rec, "occupancy")
        assert (st.voxel_visits, st.segments, st.region_misses) == \
            (ost["voxel_visits"], ost["segments"], 0)
    assert set(vm.regions) == set(om.region_keys())
    for rk, region in vm.regions.items():
        for name in names:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  om.layer(rk, name).view(np.uint8)), (rk, name)


@pytest.mark.slow
def test_c2_sequence_at_0p1m_pipelined_bit_exact():
    """The north_star target's case -- C2's OS1-128 sequence at 0.1 m voxels,
    where sample voxels collect hundreds to thousands of records per batch
    (the warp and block bucket folds) -- 10 batches through submit_batches
    against the C oracle, bit for bit."""
    from paper_2206_06079_b200 import submit_batches
    cfg = MapConfig(voxel_size=0.1)
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(100)))[:10]
    names = MODE_LAYERS["occupancy"]
    vm = VoxelMap(cfg, names)
    om = orc.OracleMap(cfg, names)
    sts = submit_batches(vm, data, "occupancy")
    for st, rec in zip(sts, data):
        ost = om.integrate_records(rec, "occupancy")
        assert (st.voxel_visits, st.segments, st.region_misses) == \
            (ost["voxel_visits"], ost["segments"], 0)
    assert max(s.records for s in sts) > 0
    assert set(vm.regions) == set(om.region_keys())
    for rk, region in vm.regions.items():
        for name in names:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  om.layer(rk, name).view(np.uint8)), (rk, name)


def _layers_equal(a, b):
    assert set(a.regions) == set(b.regions)
    for rk, region in a.regions.items():
        for name in a.layer_names:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  b.regions[rk].buffers[name].view(np.uint8)), (rk, name)


STAT_FIELDS = ("rays_in", "rays_processed", "segments", "voxel_visits", "cas_retries",
               "region_misses", "regions_touched", "records", "marked_voxels", "new_regions")


def _batches_vs_single(batches, cfg, **kw):
    from paper_2206_06079_b200 import submit_batches
    names = MODE_LAYERS["occupancy"]
    a = VoxelMap(cfg, names, **kw)
    b = VoxelMap(cfg, names, **kw)
    sa = submit_batches(a, batches, "occupancy")
    sb = [submit_batch(b, x, "occupancy") for x in batches]
    for i, (x, y) in enumerate(zip(sa, sb)):
        gx = {k: getattr(x, k) for k in STAT_FIELDS}
        gy = {k: getattr(y, k) for k in STAT_FIELDS}
        assert gx == gy, (i, {k: (gx[k], gy[k]) for k in STAT_FIELDS if gx[k] != gy[k]})
    _layers_equal(a, b)
    return sa, a


def test_submit_batches_matches_per_batch_with_pool_replays():
    """The pipelined sequence (vm_integrate_many) grows the region pool
    mid-sequence (tiny initial pool) and must equal one call per batch."""
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(40)))[:4]
    empty = data[0][:0]
    sa, _ = _batches_vs_single([data[0], empty, data[1], data[2], data[3]],
                            MapConfig(voxel_size=0.05), initial_regions=64)
    assert any(s.replays for s in sa)


def test_submit_batches_record_overflow(monkeypatch):
    """Records overflowing mid-sequence stop the chain at that batch; it is
    re-emitted and folded, the rest re-enqueued -- same result."""
    monkeypatch.setenv("VOXMAP_B200_TEST_REC_CAP", "2000")
    rng = np.random.default_rng(5)
    target = W0 + np.array([3.05, 2.05, 1.05])
    batches = [_hot_voxel_batch(rng, 300, 3000, target) for _ in range(4)]
    sa, vm = _batches_vs_single(batches, MapConfig())
    monkeypatch.delenv("VOXMAP_B200_TEST_REC_CAP")
    assert max(s.records for s in sa) > 2000
    om = orc.OracleMap(MapConfig(), MODE_LAYERS["occupancy"])
    for x in batches:
        om.integrate_records(x)
    for rk, region in vm.regions.items():
        for name in vm.layer_names:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  om.layer(rk, name).view(np.uint8)), (rk, name)


@pytest.mark.slow
def test_tsdf_then_decay_vs_oracle():
    """The C4 pattern (test_acceptance.py:398-399): per batch a TSDF pass then
    a decay pass over a map holding both layer sets, at 0.05 m."""
    cfg = MapConfig(voxel_size=0.05)
    names = tuple(dict.fromkeys(MODE_LAYERS["tsdf"] + MODE_LAYERS["decay"]))
    vm = VoxelMap(cfg, names)
    om = orc.OracleMap(cfg, names)
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(20)))[:2]
    for rec in data:
        for mode in ("tsdf", "decay"):
            st = submit_batch(vm, rec, mode, ExecutorOptions(deterministic=True))
            ost = om.integrate_records(rec, mode)
            assert st.voxel_visits == ost["voxel_visits"] and st.region_misses == 0
    assert set(vm.regions) == set(om.region_keys())
    for rk, region in vm.regions.items():
        for name in names:
            a, b = region.buffers[name], om.layer(rk, name)
            if name == "decay_distance":
                assert np.max(np.abs(a - b), initial=0.0) <= 1e-9, rk
            else:  # occupancy, mean, mean_count, decay_hits, tsdf: bit-exact
                assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (rk, name)


@pytest.mark.slow
def test_submit_batches_ndt_prefetched_matches_per_batch():
    """Non-pipelined modes run one vm_integrate per batch inside
    vm_integrate_many, with the next batch's host records prefetched into a
    device ring while the current one computes: same stats, same map."""
    from paper_2206_06079_b200 import submit_batches
    data = scans.os64_tunnel_scans(4)
    names = MODE_LAYERS["ndt-om"]
    a = VoxelMap(MapConfig(), names)
    b = VoxelMap(MapConfig(), names)
    sa = submit_batches(a, data, "ndt-om")
    sb = [submit_batch(b, x, "ndt-om") for x in data]
    for x, y in zip(sa, sb):
        assert (x.rays_processed, x.segments, x.voxel_visits, x.region_misses) == \
            (y.rays_processed, y.segments, y.voxel_visits, y.region_misses)
    assert set(a.regions) == set(b.regions)
    for rk, region in a.regions.items():
        for name in names:
            u = region.buffers[name].astype(np.float64)
            v = b.regions[rk].buffers[name].astype(np.float64)
            assert np.array_equal(u, v), (rk, name)


@pytest.mark.slow
def test_c4_uav_tsdf_then_decay_prefix_vs_oracle():
    """configs[3] (C4): the UAV lawnmower scans at 0.05 m, per batch a TSDF
    pass then a decay pass over one map holding both layer sets
    (test_acceptance.py:398-399); two scans (262k rays).  tsdf, occupancy,
    mean, mean_count and decay_hits bit-exact, decay_distance within 1e-9
    (f64 REDs, test_engine.py:56-58)."""
    cfg = MapConfig(voxel_size=0.05)
    names = tuple(dict.fromkeys(MODE_LAYERS["tsdf"] + MODE_LAYERS["decay"]))
    vm = VoxelMap(cfg, names)
    om = orc.OracleMap(cfg, names)
    for rec in scans.uav_lawnmower_scans(2):
        for mode in ("tsdf", "decay"):
            st = submit_batch(vm, rec, mode, ExecutorOptions(deterministic=True))
            ost = om.integrate_records(rec, mode)
            assert (st.voxel_visits, st.segments) == (ost["voxel_visits"], ost["segments"])
            assert st.region_misses == 0
    assert set(vm.regions) == set(om.region_keys())
    for rk, region in vm.regions.items():
        for name in names:
            a, b = region.buffers[name], om.layer(rk, name)
            if name == "decay_distance":
                assert np.max(np.abs(a - b), initial=0.0) <= 1e-9, rk
            else:
                assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (rk, name)


@pytest.mark.slow
def test_c5_town_ndt_om_prefix_bit_exact():
    """configs[4] (C5) on one GPU: town scans from the start of the drive and
    from a corner 1.5 km in (the sequence regenerates from any scan), NDT-OM
    at 0.1 m, bit-exact to the C oracle on every layer."""
    data = scans.town_scans(0, 3) + scans.town_scans(2400, 2)
    names = MODE_LAYERS["ndt-om"]
    vm = VoxelMap(MapConfig(), names)
    om = orc.OracleMap(MapConfig(), names)
    for rec in data:
        st = submit_batch(vm, rec, "ndt-om", ExecutorOptions(deterministic=True))
        ost = om.integrate_records(rec, "ndt-om")
        assert (st.voxel_visits, st.segments) == (ost["voxel_visits"], ost["segments"])
        assert st.region_misses == 0
    assert set(vm.regions) == set(om.region_keys())
    for rk, region in vm.regions.items():
        for name in names:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  om.layer(rk, name).view(np.uint8)), (rk, name)

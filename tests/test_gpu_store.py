"""Region store on HBM: eviction to OHMS1 spill files and reload, OHMR1
persistence -- the reference's own store tests (test_store.py:50-125) on the
device-resident map, plus eviction under integration (a batch that reaches
a spilled region reloads it first and the map equals one never evicted)."""
import struct
import zlib

import numpy as np
import pytest

from paper_2206_06079_b200 import ExecutorOptions, MapConfig, VoxelMap, scans, submit_batch
from paper_2206_06079_b200.keys import pack_region_coord
from paper_2206_06079_b200.layers import MODE_LAYERS

pytestmark = pytest.mark.gpu

CFG = MapConfig()


def populated_map(spill_dir=None):
    vmap = VoxelMap(CFG, ("occupancy", "mean", "mean_count"), spill_dir=spill_dir)
    rng = np.random.default_rng(11)
    for rk in [(0, 0, 0), (1, 0, 0), (-1, -1, 2)]:
        region = vmap.get_or_create_region(rk)
        region.buffers["occupancy"][:] = rng.normal(size=CFG.voxels_per_region).astype(np.float32)
        region.buffers["mean"][:] = rng.integers(0, 2 ** 30, CFG.voxels_per_region, dtype=np.uint32)
        region.buffers["mean_count"][:] = rng.integers(0, 100, CFG.voxels_per_region, dtype=np.uint32)
    return vmap


def test_eviction_round_trip_bit_exact(tmp_path):
    vmap = populated_map(spill_dir=tmp_path / "spill")
    before = {rk: {n: b.copy() for n, b in r.buffers.items()} for rk, r in vmap.regions.items()}
    vmap.batch_counter = 10
    assert vmap.evict_stale_regions(age=2) == 3
    assert vmap.region_count == 0
    files = sorted((tmp_path / "spill").glob("*.bin"))
    assert len(files) == 3
    # the reference's OHMS1 layout (store.py:137-143): the file decodes with
    # nothing but struct + zlib to the region's layer bytes
    raw = (tmp_path / "spill" / "region_-1_-1_2.bin").read_bytes()
    assert raw[:5] == b"OHMS1"
    kx, ky, kz, nl = struct.unpack_from("<3q I", raw, 5)
    assert (kx, ky, kz, nl) == (-1, -1, 2, 3)
    ids = struct.unpack_from("<3I", raw, 33)
    assert ids == (1, 2, 3)
    payload = zlib.decompress(raw[45:])
    want = b"".join(before[(-1, -1, 2)][n].tobytes() for n in ("occupancy", "mean", "mean_count"))
    assert payload == want
    assert raw[45:] == zlib.compress(want, 6)
    for rk, bufs in before.items():
        region = vmap.get_region(rk)
        assert region is not None
        for name, buf in bufs.items():
            assert np.array_equal(region.buffers[name], buf)
    assert not list((tmp_path / "spill").glob("*.bin"))  # consumed on reload


def test_eviction_respects_recency(tmp_path):
    vmap = VoxelMap(CFG, spill_dir=tmp_path)
    vmap.get_or_create_region((0, 0, 0))
    vmap.batch_counter = 5
    vmap.get_or_create_region((1, 0, 0))  # fresh access
    assert vmap.evict_stale_regions(age=2) == 1
    assert (1, 0, 0) in vmap.regions


def test_eviction_without_spill_dir_raises():
    vmap = populated_map()
    vmap.batch_counter = 10
    with pytest.raises(RuntimeError):
        vmap.evict_stale_regions(age=1)


def test_save_load_save_byte_identical(tmp_path):
    vmap = populated_map()
    p1, p2 = tmp_path / "a.bin", tmp_path / "b.bin"
    vmap.save(p1)
    VoxelMap.load(p1).save(p2)
    assert p1.read_bytes() == p2.read_bytes()


def test_save_includes_spilled_regions(tmp_path):
    vmap = populated_map(spill_dir=tmp_path / "spill")
    vmap.batch_counter = 10
    vmap.evict_stale_regions(age=2)
    path = tmp_path / "map.bin"
    vmap.save(path)
    assert len(VoxelMap.load(path).regions) == 3


def test_batches_reload_spilled_regions(tmp_path):
    """A C2 drive: after every few batches the regions the sensor left behind
    are evicted; the next batches reach some of them again (the canyon is
    re-walked by the tail of every scan).  The map -- after reloading what is
    left on disk -- equals the never-evicted map bit for bit, and the
    per-batch statistics are identical."""
    cfg = MapConfig(voxel_size=0.05)
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(120)))
    names = MODE_LAYERS["occupancy"]
    a = VoxelMap(cfg, names)
    b = VoxelMap(cfg, names, spill_dir=tmp_path / "spill")
    evicted = 0
    for i, rec in enumerate(data):
        sa = submit_batch(a, rec, "occupancy")
        sb = submit_batch(b, rec, "occupancy")
        assert (sa.voxel_visits, sa.segments, sa.region_misses, sa.regions_touched) == \
            (sb.voxel_visits, sb.segments, sb.region_misses, sb.regions_touched)
        if i % 3 == 2:
            evicted += b.evict_stale_regions(age=1)
    assert evicted > 0
    b._reload_all_spilled()
    assert set(a.regions) == set(b.regions)
    for rk, region in a.regions.items():
        for name in names:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  b.regions[rk].buffers[name].view(np.uint8)), (rk, name)


def test_pipelined_sequence_reloads_spilled_regions(tmp_path):
    from paper_2206_06079_b200 import submit_batches
    cfg = MapConfig(voxel_size=0.05)
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(60)))
    names = MODE_LAYERS["occupancy"]
    a = VoxelMap(cfg, names)
    b = VoxelMap(cfg, names, spill_dir=tmp_path / "spill")
    submit_batches(a, data[:3], "occupancy")
    submit_batches(b, data[:3], "occupancy")
    b.batch_counter += 5
    assert b.evict_stale_regions(age=1) > 0  # everything: nothing was touched in 5 batches
    assert b.region_count == 0
    sa = submit_batches(a, data[3:], "occupancy")
    sb = submit_batches(b, data[3:], "occupancy")
    assert [s.voxel_visits for s in sa] == [s.voxel_visits for s in sb]
    b._reload_all_spilled()
    assert set(a.regions) == set(b.regions)
    for rk, region in a.regions.items():
        for name in names:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  b.regions[rk].buffers[name].view(np.uint8)), (rk, name)


def test_last_access_follows_prefetch():
    """Region.last_access is the last batch whose prefetch reached the region
    (engine.py:99-118 refreshes it through get_or_create_region)."""
    cfg = MapConfig(voxel_size=0.05)
    data = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(30)))
    vm = VoxelMap(cfg, MODE_LAYERS["occupancy"])
    for rec in data[:3]:
        submit_batch(vm, rec, "occupancy")
    acc = [r.last_access for r in vm.regions.values()]
    assert max(acc) == 3 and min(acc) >= 1
    # the sensor's own region is reached by every batch
    o = data[2]["origin"][0].astype(np.float64)
    rk = tuple(int(c) for c in np.floor(o / cfg.region_size))
    assert vm.regions[rk].last_access == 3
    assert pack_region_coord(rk) >= 0


def test_pipelined_ndt_sequence_reloads_spilled_regions(tmp_path):
    """An NDT-OM sequence reaching regions spilled to disk: the guard refuses
    the batch, the runtime reloads them and replays -- the never-evicted bits."""
    from paper_2206_06079_b200 import submit_batches
    cfg = MapConfig()
    data = scans.os64_tunnel_scans(6)
    names = MODE_LAYERS["ndt-om"]
    a = VoxelMap(cfg, names)
    b = VoxelMap(cfg, names, spill_dir=tmp_path / "spill")
    submit_batches(a, data[:2], "ndt-om")
    submit_batches(b, data[:2], "ndt-om")
    b.batch_counter += 5
    assert b.evict_stale_regions(age=1) > 0
    sa = submit_batches(a, data[2:], "ndt-om")
    sb = submit_batches(b, data[2:], "ndt-om")
    assert [s.voxel_visits for s in sa] == [s.voxel_visits for s in sb]
    assert any(s.replays for s in sb)
    b._reload_all_spilled()
    assert set(a.regions) == set(b.regions)
    for rk, region in a.regions.items():
        for name in names:
            assert np.array_equal(region.buffers[name].view(np.uint8),
                                  b.regions[rk].buffers[name].view(np.uint8)), (rk, name)

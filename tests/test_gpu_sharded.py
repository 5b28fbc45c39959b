"""Region-sharded integration on one GPU with G virtual
ranks: the union of the ranks' owned regions must equal the single-GPU
deterministic map -- and so the reference's sequential executor -- bit for
bit, over several batches."""
import numpy as np
import pytest

from tests._util import digest, load_cases

pytestmark = pytest.mark.gpu

from paper_2206_06079_b200 import ExecutorOptions, MapConfig, VoxelMap, scans, submit_batch  # noqa: E402
from paper_2206_06079_b200.layers import MODE_LAYERS  # noqa: E402
from paper_2206_06079_b200.sharded import (ShardedVoxelMap, gather_owned,  # noqa: E402
                                           submit_batch_virtual)

LAYERS = MODE_LAYERS["occupancy"]
CASES = [c for c in load_cases() if c["mode"] == "occupancy"]


def _sharded(cfg, batches, world, mode="occupancy"):
    smaps = [ShardedVoxelMap(cfg, r, world, device=0, mode=mode) for r in range(world)]
    stats = [submit_batch_virtual(smaps, b) for b in batches]
    return smaps, stats


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_sharded_matches_reference_golden(case, world):
    cfg = MapConfig(**case["cfg"])
    smaps, stats = _sharded(cfg, case["batches"], world)
    for j, st in enumerate(stats):
        want = case["stats"][j].tolist()  # rays_in, processed, segments, visits, ..
        assert [st.rays_in, st.rays_processed, st.segments, st.voxel_visits] == want[:4]
        assert st.region_misses == 0
    for name in LAYERS:
        bufs = gather_owned(smaps, name)
        assert sorted(bufs) == [tuple(r) for r in case["regions"].tolist()]
        assert digest(list(bufs), lambda rk: bufs[rk]) == case["digests"][name], name


def test_sharded_scan_sequence_matches_single_gpu():
    cfg = MapConfig(voxel_size=0.05)
    batches = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(30)))[:3]
    single = VoxelMap(cfg, LAYERS)
    for b in batches:
        submit_batch(single, b, "occupancy", ExecutorOptions(deterministic=True))
    smaps, stats = _sharded(cfg, batches, 4)
    assert sum(s.voxel_visits for s in stats) > 10 ** 7
    for name in LAYERS:
        bufs = gather_owned(smaps, name)
        assert set(bufs) == set(single.regions)
        for rk, buf in bufs.items():
            assert np.array_equal(buf.view(np.uint8), single.regions[rk].buffers[name].view(np.uint8)), (rk, name)


def _dist_worker(rank, world, port, batches, q, mode="occupancy", vox=0.05):
    import os

    import torch
    import torch.distributed as dist

    from paper_2206_06079_b200.sharded import submit_batch_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        smap = ShardedVoxelMap(MapConfig(voxel_size=vox), rank, world, device=0, mode=mode)
        tot = 0
        for b in batches:
            tot += submit_batch_sharded(smap, b).voxel_visits
        owned = {rk: {n: r.buffers[n].copy() for n in MODE_LAYERS[mode]}
                 for rk, r in smap.owned_regions().items()}
        q.put((rank, tot, owned))
    finally:
        dist.destroy_process_group()


def test_sharded_distributed_driver_two_processes():
    """The torch.distributed driver (submit_batch_sharded): two processes
    sharing this GPU, exchanges over gloo through host memory."""
    import socket

    import torch.multiprocessing as mp
    cfg = MapConfig(voxel_size=0.05)
    batches = scans.batch_by_period(np.concatenate(scans.os128_canyon_batches(20)))[:2]
    single = VoxelMap(cfg, LAYERS)
    visits = 0
    for b in batches:
        visits += submit_batch(single, b, "occupancy", ExecutorOptions(deterministic=True)).voxel_visits
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, batches, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    merged = {}
    for rank, tot, owned in res:
        assert tot == visits  # every rank reports the sum over ranks
        assert not set(merged) & set(owned)
        merged.update(owned)
    assert set(merged) == set(single.regions)
    for rk, layers in merged.items():
        for n in LAYERS:
            assert np.array_equal(layers[n].view(np.uint8), single.regions[rk].buffers[n].view(np.uint8))


# ---- NDT-OM: Gaussian bitmaps out, weighed ghost visits in (vm_shard_ndt.cuh)

NDT_CASES = [c for c in load_cases() if c["mode"] == "ndt-om"]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", NDT_CASES, ids=[c["name"] for c in NDT_CASES])
def test_sharded_ndt_matches_reference_golden(case, world):
    """Every NDT-OM layer of the union of owned regions has the reference's
    own digest (the single-GPU NDT path is bit-exact to it)."""
    cfg = MapConfig(**case["cfg"])
    smaps, stats = _sharded(cfg, case["batches"], world, "ndt-om")
    for j, st in enumerate(stats):
        want = case["stats"][j].tolist()
        assert [st.rays_in, st.rays_processed, st.segments, st.voxel_visits] == want[:4]
        assert st.region_misses == 0
    for name in MODE_LAYERS["ndt-om"]:
        bufs = gather_owned(smaps, name)
        assert sorted(bufs) == [tuple(r) for r in case["regions"].tolist()]
        assert digest(list(bufs), lambda rk: bufs[rk]) == case["digests"][name], name


def _single(cfg, batches, mode):
    single = VoxelMap(cfg, MODE_LAYERS[mode])
    visits = 0
    for b in batches:
        visits += submit_batch(single, b, mode, ExecutorOptions(deterministic=True)).voxel_visits
    return single, visits


def _assert_union_equals(bufs_by_name, single, names):
    for name in names:
        bufs = bufs_by_name(name)
        assert set(bufs) == set(single.regions)
        for rk, buf in bufs.items():
            assert np.array_equal(buf.view(np.uint8),
                                  single.regions[rk].buffers[name].view(np.uint8)), (rk, name)


@pytest.mark.slow
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_ndt_tunnel_scans_match_single_gpu(world):
    """Four C3 tunnel scans: from the second scan on, most misses cross
    Gaussian voxels, many of them other ranks' -- weighed by their owners."""
    cfg = MapConfig()
    batches = scans.os64_tunnel_scans(4)
    single, visits = _single(cfg, batches, "ndt-om")
    smaps, stats = _sharded(cfg, batches, world, "ndt-om")
    assert sum(s.voxel_visits for s in stats) == visits
    _assert_union_equals(lambda n: gather_owned(smaps, n), single, MODE_LAYERS["ndt-om"])


@pytest.mark.slow
def test_sharded_ndt_town_scans_match_single_gpu():
    """configs[4] (C5) -- NDT-OM over region-sharded ranks -- on a prefix:
    three town scans, 8 virtual ranks."""
    cfg = MapConfig()
    batches = scans.town_scans(0, 3)
    single, visits = _single(cfg, batches, "ndt-om")
    smaps, stats = _sharded(cfg, batches, 8, "ndt-om")
    assert sum(s.voxel_visits for s in stats) == visits
    _assert_union_equals(lambda n: gather_owned(smaps, n), single, MODE_LAYERS["ndt-om"])


def test_sharded_ndt_distributed_driver_two_processes():
    """submit_batch_sharded for NDT-OM in two processes over gloo."""
    import socket

    import torch.multiprocessing as mp
    cfg = MapConfig()
    batches = [t[::4].copy() for t in scans.os64_tunnel_scans(3)]
    single, visits = _single(cfg, batches, "ndt-om")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, batches, q, "ndt-om", 0.1))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    merged = {}
    for rank, tot, owned in res:
        assert tot == visits
        assert not set(merged) & set(owned)
        merged.update(owned)
    _assert_union_equals(lambda n: {rk: v[n] for rk, v in merged.items()}, single,
                         MODE_LAYERS["ndt-om"])

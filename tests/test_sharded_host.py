"""Host side of the region-sharded mode on CPU: the variable-size
all-to-all / all-gather used for the record exchange, the slice-upload +
all-gather of the batch (gloo, world size 2), and the region-ownership
function (vm_shard_owner, needs no device)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2206_06079_b200 import _native  # noqa: E402
from paper_2206_06079_b200.keys import pack_region_coord  # noqa: E402
from paper_2206_06079_b200.sharded import (_gather_batch, exchange_all_gather,  # noqa: E402
                                           exchange_all_to_all)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r sends (r+1)*(d+1) rows of [r, d, i] to rank d
        sends = [torch.tensor([[rank, d, i] for i in range((rank + 1) * (d + 1))], dtype=torch.int64)
                 .reshape(-1, 3) for d in range(world)]
        got = exchange_all_to_all(sends)
        rows = [g.tolist() for g in got]
        gathered = exchange_all_gather(torch.full((rank + 2, 2), rank, dtype=torch.int64))
        # the batch: each rank contributes its slice, every rank gets it whole
        from paper_2206_06079_b200 import scans
        batch = scans.os64_room_scan(seed=0)[:1001]
        full = _gather_batch(batch, "cpu", None, host=True)
        same = bool(np.array_equal(full.numpy(), batch.view(np.uint8).reshape(-1)))
        q.put((rank, rows, gathered.tolist(), same))
    finally:
        dist.destroy_process_group()


def test_variable_size_exchange_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, rows, gathered, same = q.get(timeout=120)
        res[r] = (rows, gathered)
        assert same
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        rows, gathered = res[r]
        for src in range(world):
            assert rows[src] == [[src, r, i] for i in range((src + 1) * (r + 1))]
        assert gathered == [[0, 0]] * 2 + [[1, 1]] * 3


def _owner_ref(rk, world):
    # region_owner (vm_device.cuh): splitmix64 of the packed 2x2x2 block key, mod world
    m = (1 << 64) - 1
    b = pack_region_coord(tuple(c >> 1 for c in rk))
    h = (b + 0x9E3779B97F4A7C15) & m
    h = ((h ^ (h >> 30)) * 0xBF58476D1CE4E5B9) & m
    h = ((h ^ (h >> 27)) * 0x94D049BB133111EB) & m
    return (h ^ (h >> 31)) % world


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_region_owner_blocks_and_balance(world):
    rng = np.random.default_rng(world)
    coords = rng.integers(-300, 300, (4000, 3))
    owners = np.array([_native.shard_owner(pack_region_coord(tuple(int(x) for x in c)), world)
                       for c in coords])
    assert owners.min() >= 0 and owners.max() < world
    for c, o in zip(coords[:300], owners[:300]):
        assert o == _owner_ref(tuple(int(x) for x in c), world)
        # the 2x2x2 block shares one owner
        base = tuple(int(x) & ~1 for x in c)
        assert _native.shard_owner(pack_region_coord(base), world) == o
    if world > 1:
        share = np.bincount(owners, minlength=world) / len(owners)
        assert share.min() > 0.5 / world

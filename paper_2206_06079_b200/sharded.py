"""Region-sharded integration over G GPUs.

One process per GPU (torch.distributed, NCCL over NVLink) -- or, for tests on
a single GPU, G "virtual ranks" in one process.  Rank r's map owns the regions
with `shard_owner(key, G) == r` (2 x 2 x 2 region blocks hashed over the
ranks) and walks the slice [r*N/G, (r+1)*N/G) of every batch; every rank is
handed the whole batch.  Per batch (protocol in csrc/vm_shard.cuh):

  begin / lists   discover the slice; creation requests for new regions other
                  ranks own, and the slice's new sample voxels
  exchange A      requests all-to-all, sample voxels all-gather
  prepare         create the requested regions, stamp every rank's sample voxels
  walk            the deterministic walk of the slice
  export          per-owner payload: miss counts of ghost voxels and the
                  order-keyed records of ghost sample voxels (16-byte items)
  exchange B      payload all-to-all
  import, finish  owners apply the payload, then resolve / sort / fold

NDT-OM (mode="ndt-om", csrc/vm_shard_ndt.cuh) replaces the sample-voxel
marks with Gaussian bitmaps: every rank requests the bitmaps (count >= 3 at
the start of the batch) of the ghost regions its slice prefetched, its walk
sends each visit through a ghost Gaussian voxel to the owner with the
segment order and chord (t0, t1), and the owner weighs it with its own
Gaussian -- so phase 1 is complete before any phase-2 update, as in the
reference (engine.py:285).

The union of the ranks' owned regions is the single-GPU map, bit for bit
(tests/test_gpu_sharded.py), for deterministic occupancy and NDT-OM.
"""
from __future__ import annotations

import numpy as np

from . import _native
from .engine import BatchStats
from .keys import unpack_region_coord
from .layers import MODE_LAYERS
from .store import VoxelMap

ITEM_WORDS = 2      # a 16-byte ShardItem as two int64
ITEM_WORDS_NDT = 4  # a 32-byte ShardItemN (NDT-OM) as four int64


def _torch():
    import torch
    return torch


_STREAMS: dict = {}


def _shared_stream(device: int):
    """The sharded maps' stream on `device` (virtual ranks on one device share
    it, so their exchanges and kernels are totally ordered)."""
    torch = _torch()
    if device not in _STREAMS:
        _STREAMS[device] = torch.cuda.Stream(device=device)
    return _STREAMS[device]


class ShardedVoxelMap:
    """This rank's part of a region-sharded map."""

    def __init__(self, cfg, rank: int, world: int, device: int = 0,
                 layer_names=None, initial_regions: int = 1024, mode: str = "occupancy"):
        if mode not in ("occupancy", "ndt-om"):
            raise ValueError("sharded maps integrate deterministic occupancy or NDT-OM")
        self.mode = mode
        layer_names = MODE_LAYERS[mode] if layer_names is None else layer_names
        self.cfg = cfg
        self.rank, self.world, self.device = int(rank), int(world), int(device)
        self.vmap = VoxelMap(cfg, layer_names, device=self.device, initial_regions=initial_regions)
        self.nat = self.vmap._native
        self.nat.shard_config(self.rank, self.world)
        # One explicit stream per device, shared by this map's kernels and by
        # every torch op of the exchange (the drivers below run them under
        # `torch.cuda.stream(self.stream)`; NCCL collectives are ordered
        # against the current stream).  Never torch's legacy default stream:
        # its handle is 0, which the runtime would read as "create a private
        # non-blocking stream" with no ordering against torch's work.
        self.stream = _shared_stream(self.device)
        self.nat.set_stream(self.stream.cuda_stream)
        self._keep = None
        self._cap = 1 << 16  # export items per destination

    @property
    def dev(self):
        return _torch().device("cuda", self.device)

    def owned_regions(self) -> dict:
        """{region coord: Region} of the regions this rank owns."""
        self.vmap._sync_regions()
        return {rk: r for rk, r in self.vmap.regions.items()
                if _native.shard_owner(self._packed(rk), self.world) == self.rank}

    @staticmethod
    def _packed(rk) -> int:
        B, M = 1 << 20, (1 << 21) - 1
        return ((rk[0] + B) & M) << 42 | ((rk[1] + B) & M) << 21 | ((rk[2] + B) & M)

    # ---- phases -------------------------------------------------------

    def begin(self, records_dev):
        """records_dev: uint8 device tensor of the whole batch (OHMB1)."""
        torch = _torch()
        rays = _native.rays_from_records(records_dev.numel() // 40, records_dev.data_ptr())
        self._keep = records_dev
        self.vmap.flush_host_writes()
        self.vmap.batch_counter += 1
        self.vmap._begin_batch()
        nnew, nmarks = self.nat.shard_begin(rays, self.mode)
        req = torch.empty((self.world, max(nnew, 1)), dtype=torch.int64, device=self.dev)
        marks = torch.empty((max(nmarks, 1), 2), dtype=torch.int64, device=self.dev)
        counts = self.nat.shard_lists(req.data_ptr(), req.shape[1], marks.data_ptr(), marks.shape[0],
                                      self.world)
        sends = [req[d, :counts[1 + d]] for d in range(self.world)]
        return sends, marks[:counts[0]]

    # ---- NDT-OM: Gaussian bitmaps of the ghost regions ------------------

    @property
    def bit_words(self) -> int:
        return (self.cfg.region_dim ** 3 + 31) // 32

    def ndt_bits(self, req_in):
        """Owner side: the bitmaps of the regions other ranks requested
        (int32 [n, words] device tensor, in request order)."""
        torch = _torch()
        req_in = req_in.contiguous()
        out = torch.empty((max(req_in.numel(), 1), self.bit_words), dtype=torch.int32, device=self.dev)
        self.nat.shard_ndt_bits(req_in.data_ptr(), req_in.numel(), out.data_ptr())
        return out[:req_in.numel()]

    def ndt_mark(self, keys, bits):
        keys = keys.contiguous()
        bits = bits.contiguous()
        self.nat.shard_ndt_mark(keys.data_ptr(), bits.data_ptr(), keys.numel())

    def prepare(self, req_in, marks_all):
        req_in = req_in.contiguous()
        marks_all = marks_all.contiguous()
        self.nat.shard_prepare(req_in.data_ptr(), req_in.numel(), marks_all.data_ptr(),
                               marks_all.shape[0])

    def walk(self):
        self.nat.shard_walk()

    def export(self):
        torch = _torch()
        words = ITEM_WORDS if self.mode == "occupancy" else ITEM_WORDS_NDT
        while True:
            out = torch.empty((self.world, self._cap, words), dtype=torch.int64, device=self.dev)
            rc, counts = self.nat.shard_export(out.data_ptr(), self._cap, self.world)
            if rc == _native.VM_OK:
                return [out[d, :counts[d]] for d in range(self.world)]
            if rc != _native.VM_ERR_ARG or max(counts) <= self._cap:
                _native.check(rc, "vm_shard_export")
            self._cap = 1 << int(max(counts) - 1).bit_length()

    def import_(self, items):
        items = items.contiguous()
        self.nat.shard_import(items.data_ptr(), items.shape[0])

    def finish(self) -> BatchStats:
        st = self.nat.shard_finish()
        self.vmap._sync_regions()
        self._keep = None
        return BatchStats(rays_in=int(st.rays_in), rays_processed=int(st.rays_processed),
                          segments=int(st.segments), voxel_visits=int(st.voxel_visits),
                          region_misses=int(st.region_misses),
                          regions_touched=int(st.regions_touched), gpu_time=st.gpu_ms * 1e-3,
                          walk_time=st.walk_ms * 1e-3, records=int(st.records))


def _sum_stats(parts) -> BatchStats:
    out = BatchStats()
    for s in parts:
        for f in ("rays_in", "rays_processed", "segments", "voxel_visits", "region_misses",
                  "records"):
            setattr(out, f, getattr(out, f) + getattr(s, f))
        out.gpu_time = max(out.gpu_time, s.gpu_time)
        out.walk_time = max(out.walk_time, s.walk_time)
    return out


def _to_device(records, dev):
    torch = _torch()
    if isinstance(records, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(records).view(np.uint8).reshape(-1)).to(dev)
    return records.to(dev)


# ---- one process per GPU (torch.distributed) ----------------------------

def _gather_batch(records, dev, group, host: bool):
    """The whole batch on this rank's device.  Host records: every rank
    uploads only its own slice [r*N/G, (r+1)*N/G) and the slices are
    all-gathered device to device (NVLink with NCCL), instead of each rank
    copying the whole batch over PCIe.  Device records are used as they are."""
    torch = _torch()
    import torch.distributed as dist
    if not isinstance(records, np.ndarray):
        return records.to(dev)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    rec = np.ascontiguousarray(records).view(np.uint8).reshape(-1, 40)
    n = rec.shape[0]
    per = (n + world - 1) // world
    lo, hi = n * rank // world, n * (rank + 1) // world
    mine = torch.zeros((per, 40), dtype=torch.uint8)
    mine[:hi - lo] = torch.from_numpy(rec[lo:hi])
    mine = mine if host else mine.to(dev)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    full = torch.cat([p[:n * (q + 1) // world - n * q // world] for q, p in enumerate(parts)])
    return full.reshape(-1).to(dev)


def exchange_all_to_all(sends, group=None):
    """Variable-size all-to-all of 1-D/2-D tensors (same trailing shape):
    sends[d] goes to rank d; returns the tensors received from each rank.
    NCCL for CUDA tensors, gloo for CPU tensors."""
    torch = _torch()
    import torch.distributed as dist
    world = len(sends)
    dev = sends[0].device
    tail = tuple(sends[0].shape[1:])
    cnt_out = torch.tensor([s.shape[0] for s in sends], dtype=torch.int64, device=dev)
    cnt_in = torch.empty_like(cnt_out)
    dist.all_to_all_single(cnt_in, cnt_out, group=group)
    rin = [int(x) for x in cnt_in.cpu()]
    send = torch.cat([s.reshape(-1, *tail) for s in sends]) if world else sends[0]
    recv = torch.empty((sum(rin),) + tail, dtype=send.dtype, device=dev)
    dist.all_to_all_single(recv, send, output_split_sizes=rin,
                           input_split_sizes=[s.shape[0] for s in sends], group=group)
    return list(torch.split(recv, rin))


def exchange_all_gather(t, group=None):
    """Variable-size all-gather along dim 0."""
    torch = _torch()
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    ns = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    sizes = [int(x.item()) for x in ns]
    mx = max(sizes + [1])
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[:t.shape[0]] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:s] for o, s in zip(outs, sizes)])


def submit_batch_sharded(smap: ShardedVoxelMap, records, group=None) -> BatchStats:
    """Integrate one batch into this rank's part of a region-sharded map
    (collective over `group`); see _submit_sharded."""
    with _torch().cuda.stream(smap.stream):
        return _submit_sharded(smap, records, group)


def _submit_sharded(smap: ShardedVoxelMap, records, group=None) -> BatchStats:
    """Integrate one batch (the whole batch on every rank) into this rank's
    part of the map; collective over `group` (NCCL: device buffers go
    straight over NVLink; gloo: staged through host memory, for CPU-side
    tests of the protocol).  Returns the batch statistics summed over the
    ranks."""
    torch = _torch()
    import torch.distributed as dist
    host = dist.get_backend(group) == "gloo"
    dev = smap.dev
    wire = (lambda t: t.cpu()) if host else (lambda t: t)
    rec = _gather_batch(records, dev, group, host)
    sends, marks = smap.begin(rec)
    if smap.mode == "ndt-om":
        # requests out, Gaussian bitmaps back (in request order), then mark
        got = exchange_all_to_all([wire(t) for t in sends], group)
        answers = [smap.ndt_bits(t.to(dev)) for t in got]
        back = exchange_all_to_all([wire(a) for a in answers], group)
        smap.ndt_mark(torch.cat(sends), torch.cat([b.to(dev) for b in back]))
        answered = sum(int(a.numel() * a.element_size()) for r, a in enumerate(answers)
                       if r != dist.get_rank(group))
    else:
        req_in = torch.cat(exchange_all_to_all([wire(t) for t in sends], group)).to(dev)
        smap.prepare(req_in, exchange_all_gather(wire(marks), group).to(dev))
        answered = 0
    smap.walk()
    exported = smap.export()
    items = torch.cat(exchange_all_to_all([wire(t) for t in exported], group)).to(dev)
    smap.import_(items)
    st = smap.finish()
    # bytes this rank sent to other ranks (requests, sample-voxel marks to
    # every peer, counts / records to their owners)
    me = dist.get_rank(group)
    world = dist.get_world_size(group)
    sent = sum(int(t.numel() * t.element_size()) for r, t in enumerate(sends) if r != me)
    sent += int(marks.numel() * marks.element_size()) * (world - 1)
    sent += sum(int(t.numel() * t.element_size()) for r, t in enumerate(exported) if r != me)
    sent += answered
    v = torch.tensor([st.rays_in, st.rays_processed, st.segments, st.voxel_visits,
                      st.region_misses, st.records, sent], dtype=torch.int64,
                     device="cpu" if host else dev)
    dist.all_reduce(v, group=group)
    (st.rays_in, st.rays_processed, st.segments, st.voxel_visits, st.region_misses,
     st.records, st.exchange_bytes) = [int(x) for x in v.cpu()]
    return st


# ---- virtual ranks in one process (tests, single-GPU boxes) -------------

def submit_batch_virtual(smaps, records) -> BatchStats:
    """The same protocol for G ShardedVoxelMaps living in this process (any
    devices); the exchanges are device copies."""
    import contextlib
    torch = _torch()
    with contextlib.ExitStack() as stack:
        # every device's current stream is its maps' stream (torch orders
        # cross-device copies against the current streams of both devices)
        for st in {s.device: s.stream for s in smaps}.values():
            stack.enter_context(torch.cuda.stream(st))
        return _submit_virtual(smaps, records)


def _submit_virtual(smaps, records) -> BatchStats:
    torch = _torch()
    world = len(smaps)
    recs = [_to_device(records, s.dev) for s in smaps]
    begun = [s.begin(r) for s, r in zip(smaps, recs)]
    if smaps[0].mode == "ndt-om":
        # answers[r][q]: rank r's bitmaps for rank q's requests
        answers = [[s.ndt_bits(begun[q][0][r].to(s.dev)) for q in range(world)]
                   for r, s in enumerate(smaps)]
        for q, s in enumerate(smaps):
            keys = torch.cat([begun[q][0][r] for r in range(world)])
            bits = torch.cat([answers[r][q].to(s.dev) for r in range(world)])
            s.ndt_mark(keys, bits)
    else:
        marks_all = [torch.cat([m.to(s.dev) for _, m in begun]) for s in smaps]
        for r, s in enumerate(smaps):
            req_in = torch.cat([begun[q][0][r].to(s.dev) for q in range(world)])
            s.prepare(req_in, marks_all[r])
    for s in smaps:
        s.walk()
    exports = [s.export() for s in smaps]
    for r, s in enumerate(smaps):
        s.import_(torch.cat([exports[q][r].to(s.dev) for q in range(world)]))
    return _sum_stats([s.finish() for s in smaps])


def gather_owned(smaps, layer: str) -> dict:
    """{region coord: host buffer of `layer`} over every rank's owned regions."""
    out = {}
    for s in smaps:
        for rk, region in s.owned_regions().items():
            out[rk] = region.buffers[layer]
    return out


__all__ = ["ShardedVoxelMap", "submit_batch_sharded", "submit_batch_virtual", "gather_owned",
           "exchange_all_to_all", "exchange_all_gather", "unpack_region_coord"]

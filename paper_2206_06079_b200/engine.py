"""Batch integration entry point (mirror of voxmap.engine, engine.py:26-216).

`submit_batch` hands the whole batch to the CUDA runtime in one call
(vm_integrate): clip + segment, region prefetch, DDA walk and layer updates
all run on the GPU.  There is no CPU executor and no fallback.

Executors map onto the two device update paths:

* deterministic (`ExecutorOptions(kind="sequential")`, and the default
  single-worker `kind="parallel"`): order-free misses are counted and
  resolved as f_miss^k, visits to sample voxels are emitted as
  (voxel, ray order, hit) records, radix-sorted and folded in ray order.
  Results are bit-identical to the reference's sequential executor
  (engine.py:213-237) for occupancy, mean, mean_count, decay_hits and tsdf.
* CAS (`kind="parallel"` with worker_count > 1, or `deterministic=False`):
  the paper's lock-free compare-and-swap update (_kernels.pyx:233-357);
  order-dependent only on voxels that receive both hits and misses.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native
from . import layers
from .rayset import RAY_DTYPE, RayBatch
from .store import VoxelMap

MODES = tuple(layers.MODE_LAYERS)


class ConfigurationError(Exception):
    """Map layers do not match what the requested integrator needs."""


@dataclass
class BatchStats:
    rays_in: int = 0
    rays_processed: int = 0
    segments: int = 0
    voxel_visits: int = 0
    cas_retries: int = 0
    cas_failures: int = 0
    region_misses: int = 0
    regions_touched: int = 0
    wall_time: float = 0.0
    # device-side extras
    gpu_time: float = 0.0
    walk_time: float = 0.0
    records: int = 0
    marked_voxels: int = 0
    new_regions: int = 0
    replays: int = 0
    exchange_bytes: int = 0  # region-sharded maps: bytes sent between ranks, all ranks

    @property
    def rays_per_second(self) -> float:
        if self.wall_time <= 0.0:
            return 0.0
        return self.rays_processed / self.wall_time

    def csv_row(self) -> str:
        return ",".join(str(v) for v in (
            self.rays_in, self.rays_processed, self.segments, self.voxel_visits,
            self.cas_retries, self.cas_failures, f"{self.wall_time:.6f}",
            f"{self.rays_per_second:.1f}"))


@dataclass
class ExecutorOptions:
    worker_count: int = 1
    cas_retry_limit: int = 20
    kind: str = "parallel"
    deterministic: bool | None = None

    def __post_init__(self):
        if self.worker_count < 1:
            raise ValueError("worker_count must be >= 1")
        if self.kind not in ("sequential", "parallel"):
            raise ValueError(f"unknown executor kind {self.kind!r}")
        if self.kind == "sequential" and self.worker_count != 1:
            raise ValueError("sequential executor requires worker_count == 1")
        if self.kind == "sequential" and self.deterministic is False:
            raise ValueError("the sequential executor is deterministic")

    @property
    def use_deterministic(self) -> bool:
        if self.deterministic is not None:
            return bool(self.deterministic)
        return self.kind == "sequential" or self.worker_count == 1


def _as_native_rays(rays):
    """list[RaySample] | OHMB1 record array | RayBatch -> (VmRays, keepalive)."""
    if isinstance(rays, np.ndarray) and rays.dtype == RAY_DTYPE:
        rec = np.ascontiguousarray(rays)
        return _native.rays_from_records(rec), rec
    if isinstance(rays, RayBatch):
        return _native.rays_from_arrays(rays.origins, rays.ends, rays.has_sample, rays.intensity)
    batch = RayBatch.from_samples(list(rays))
    return _native.rays_from_arrays(batch.origins, batch.ends, batch.has_sample, batch.intensity)


def submit_batch(vmap: VoxelMap, rays, mode: str, opts: ExecutorOptions | None = None
                 ) -> BatchStats:
    """Integrate one batch of rays with the given integrator mode (engine.py:175-210)."""
    if opts is None:
        opts = ExecutorOptions()
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {MODES}")
    required = layers.MODE_LAYERS[mode]
    if not vmap.has_layers(required):
        missing = set(required) - set(vmap.layer_names)
        raise ConfigurationError(f"map lacks layers {sorted(missing)} required by mode {mode!r}")
    start = time.perf_counter()
    native_rays, keep = _as_native_rays(rays)
    stats = BatchStats(rays_in=int(native_rays.count))
    vmap.batch_counter += 1
    vmap.flush_host_writes()
    vmap._begin_batch()
    st = vmap._native.integrate(native_rays, mode, opts.use_deterministic)
    del keep
    vmap._note_batch(int(st.regions_total))
    stats.rays_processed = int(st.rays_processed)
    stats.segments = int(st.segments)
    stats.voxel_visits = int(st.voxel_visits)
    stats.cas_retries = int(st.cas_retries)
    stats.cas_failures = int(st.cas_failures)
    stats.region_misses = int(st.region_misses)
    stats.regions_touched = int(st.regions_touched)
    stats.gpu_time = float(st.gpu_ms) * 1e-3
    stats.walk_time = float(st.walk_ms) * 1e-3
    stats.records = int(st.records)
    stats.marked_voxels = int(st.marked_voxels)
    stats.new_regions = int(st.new_regions)
    stats.replays = int(st.replays)
    stats.wall_time = time.perf_counter() - start
    return stats


def _to_stats(st, wall: float) -> BatchStats:
    stats = BatchStats(rays_in=int(st.rays_in))
    for name in ("rays_processed", "segments", "voxel_visits", "cas_retries", "cas_failures",
                 "region_misses", "regions_touched", "records", "marked_voxels", "new_regions",
                 "replays"):
        setattr(stats, name, int(getattr(st, name)))
    stats.gpu_time = float(st.gpu_ms) * 1e-3
    stats.walk_time = float(st.walk_ms) * 1e-3
    stats.wall_time = wall
    return stats


def submit_batches(vmap: VoxelMap, batches, mode: str, opts: ExecutorOptions | None = None
                   ) -> list[BatchStats]:
    """Integrate a sequence of batches in order: the same map state and the
    same per-batch stats as calling `submit_batch` once per batch (the
    reference CLI's offline replay loop, cli.py:122-127).  Deterministic
    occupancy and NDT over OHMB1 record arrays run as one pipelined device sequence
    (vm_integrate_many: host uploads overlap earlier batches' compute, one
    sync at the end); `wall_time` of each batch is its share of the call."""
    if opts is None:
        opts = ExecutorOptions()
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {MODES}")
    required = layers.MODE_LAYERS[mode]
    if not vmap.has_layers(required):
        missing = set(required) - set(vmap.layer_names)
        raise ConfigurationError(f"map lacks layers {sorted(missing)} required by mode {mode!r}")
    batches = list(batches)
    if not batches:
        return []
    start = time.perf_counter()
    converted = [_as_native_rays(b) for b in batches]
    vmap.batch_counter += 1  # the sequence's first batch; the device counts on
    vmap.flush_host_writes()
    vmap._begin_batch()
    sts = vmap._native.integrate_many([c[0] for c in converted], mode, opts.use_deterministic)
    del converted
    vmap.batch_counter += len(batches) - 1
    vmap._note_batch(int(sts[-1].regions_total))
    wall = time.perf_counter() - start
    total = sum(int(s.rays_in) for s in sts) or 1
    return [_to_stats(s, wall * int(s.rays_in) / total) for s in sts]


def sequential_reference(vmap: VoxelMap, rays, mode: str = "occupancy") -> BatchStats:
    """Deterministic executor: the reference's sequential results, on the GPU."""
    return submit_batch(vmap, rays, mode, ExecutorOptions(worker_count=1, kind="sequential"))

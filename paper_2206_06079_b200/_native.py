"""ctypes binding of the C ABI in include/voxmap_b200.h.

This is the only way the package reaches the hot path: there is no Python
or CPU fallback.  If the in-tree library is missing or no CUDA device is
present, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import math
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libvoxmap_b200.so"

VM_OK, VM_ERR_ARG, VM_ERR_CUDA, VM_ERR_OOM, VM_ERR_RANGE, VM_ERR_NODEV = range(6)
MODES = ("occupancy", "decay", "ndt-om", "ndt-tm", "tsdf")
EXEC_CAS, EXEC_DETERMINISTIC = 0, 1
RAYS_OHMB1, RAYS_F64 = 0, 1
I64_t = ctypes.c_int64

EXPORTED = (
    "vm_map_create", "vm_map_destroy", "vm_map_reset", "vm_map_set_stream", "vm_map_region_count",
    "vm_map_set_batch_counter", "vm_map_region_last_access", "vm_map_set_spill",
    "vm_map_evict_regions", "vm_map_reload_region", "vm_map_spilled_keys",
    "vm_map_region_keys", "vm_map_ensure_regions", "vm_map_find_region", "vm_map_read_layer",
    "vm_map_write_layer", "vm_map_layer_ptr", "vm_integrate", "vm_integrate_many", "vm_export_select", "vm_export_gather", "vm_walk_voxels", "vm_ndt_hypot", "vm_hash_mix",
    "vm_kernels_integrate_occupancy", "vm_last_error", "vm_device_count", "vm_build_info",
    "vm_shard_config", "vm_shard_owner", "vm_shard_begin", "vm_shard_lists", "vm_shard_prepare",
    "vm_shard_walk", "vm_shard_ndt_bits", "vm_shard_ndt_mark",
    "vm_shard_export", "vm_shard_import", "vm_shard_finish", "vm_probe_red_rate",
)


class NativeError(RuntimeError):
    pass


class NoDeviceError(NativeError):
    pass


class VmConfig(ctypes.Structure):
    _fields_ = [
        ("voxel_size", ctypes.c_double), ("region_dim", ctypes.c_int32), ("_pad", ctypes.c_int32),
        ("hit_delta", ctypes.c_double), ("miss_delta", ctypes.c_double),
        ("clamp_min", ctypes.c_double), ("clamp_max", ctypes.c_double),
        ("max_ray_range", ctypes.c_double), ("segment_length", ctypes.c_double),
        ("tsdf_truncation", ctypes.c_double), ("tsdf_max_weight", ctypes.c_double),
        ("ndt_sensor_noise", ctypes.c_double), ("ndt_reset_threshold", ctypes.c_double),
        ("ndt_miss_likelihood_threshold", ctypes.c_double),
    ]


class VmStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "rays_in", "rays_processed", "segments", "voxel_visits", "cas_retries", "cas_failures",
        "region_misses", "regions_touched", "records", "marked_voxels", "regions_total",
        "new_regions", "replays", "touched_regions_walk", "launches")] + [
        ("gpu_ms", ctypes.c_double), ("walk_ms", ctypes.c_double),
        ("discover_ms", ctypes.c_double), ("resolve_ms", ctypes.c_double),
        ("sort_ms", ctypes.c_double), ("fold_ms", ctypes.c_double)]


class VmRays(ctypes.Structure):
    _fields_ = [
        ("format", ctypes.c_int32), ("on_device", ctypes.c_int32), ("count", ctypes.c_int64),
        ("records", ctypes.c_void_p), ("origins", ctypes.c_void_p), ("ends", ctypes.c_void_p),
        ("has_sample", ctypes.c_void_p), ("intensity", ctypes.c_void_p),
    ]


_lib = None


def lib():
    """Load the in-tree CUDA library (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = LIB_PATH
    if os.environ.get("VOXMAP_B200_LIB"):  # dev knob: an in-tree build variant (tools/variants)
        path = LIB_PATH.parent / os.environ["VOXMAP_B200_LIB"]
    if not path.exists():
        raise NativeError(
            f"CUDA extension not built: {path} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
    L = ctypes.CDLL(str(path))
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "vm_map_create": ([ctypes.POINTER(VmConfig), ctypes.c_uint32, I32, I64,
                           ctypes.POINTER(P)], ctypes.c_int),
        "vm_map_destroy": ([P], ctypes.c_int),
        "vm_map_reset": ([P], ctypes.c_int),
        "vm_map_set_stream": ([P, P], ctypes.c_int),
        "vm_map_region_count": ([P, ctypes.POINTER(I64)], ctypes.c_int),
        "vm_map_region_keys": ([P, I64, I64, P], ctypes.c_int),
        "vm_map_ensure_regions": ([P, P, I64, P], ctypes.c_int),
        "vm_map_find_region": ([P, I64, ctypes.POINTER(I32)], ctypes.c_int),
        "vm_map_read_layer": ([P, I32, I32, P, I64], ctypes.c_int),
        "vm_map_write_layer": ([P, I32, I32, P, I64], ctypes.c_int),
        "vm_map_layer_ptr": ([P, I32, I32, ctypes.POINTER(P)], ctypes.c_int),
        "vm_integrate": ([P, ctypes.POINTER(VmRays), I32, I32, ctypes.POINTER(VmStats)],
                         ctypes.c_int),
        "vm_integrate_many": ([P, ctypes.POINTER(VmRays), I32, I32, I32, ctypes.POINTER(VmStats)],
                              ctypes.c_int),
        "vm_export_select": ([P, P, I64, I32, D, ctypes.POINTER(I64), P, P, I64], ctypes.c_int),
        "vm_export_gather": ([P, I32, P, I64, P, P, I64, P], ctypes.c_int),
        "vm_walk_voxels": ([D] * 7 + [I64, P, P, P, ctypes.POINTER(I64)], ctypes.c_int),
        "vm_ndt_hypot": ([P, I64, P], ctypes.c_int),
        "vm_hash_mix": ([I64], ctypes.c_uint64),
        "vm_kernels_integrate_occupancy": ([P, P, P, I64, P, P, I64, P, P, P, P, P, D, I64, D, D,
                                            D, D, I32, I32, P, P], ctypes.c_int),
        "vm_last_error": ([], ctypes.c_char_p),
        "vm_shard_config": ([P, I32, I32], ctypes.c_int),
        "vm_shard_owner": ([I64, I32], ctypes.c_int),
        "vm_shard_begin": ([P, ctypes.POINTER(VmRays), I32, I32, P], ctypes.c_int),
        "vm_shard_lists": ([P, P, I64, P, I64, P], ctypes.c_int),
        "vm_shard_prepare": ([P, P, I64, P, I64], ctypes.c_int),
        "vm_shard_walk": ([P], ctypes.c_int),
        "vm_shard_ndt_bits": ([P, P, I64, P], ctypes.c_int),
        "vm_shard_ndt_mark": ([P, P, P, I64], ctypes.c_int),
        "vm_shard_export": ([P, P, I64, P], ctypes.c_int),
        "vm_shard_import": ([P, P, I64], ctypes.c_int),
        "vm_shard_finish": ([P, ctypes.POINTER(VmStats)], ctypes.c_int),
        "vm_device_count": ([ctypes.POINTER(I32)], ctypes.c_int),
        "vm_build_info": ([], ctypes.c_char_p),
        "vm_probe_red_rate": ([I32, I64, I32, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "vm_map_set_batch_counter": ([P, ctypes.c_uint32], ctypes.c_int),
        "vm_map_region_last_access": ([P, I64, I64, P], ctypes.c_int),
        "vm_map_set_spill": ([P, ctypes.c_char_p, P, I32], ctypes.c_int),
        "vm_map_evict_regions": ([P, P, I64, P], ctypes.c_int),
        "vm_map_reload_region": ([P, I64, ctypes.POINTER(I32)], ctypes.c_int),
        "vm_map_spilled_keys": ([P, P, I64, P], ctypes.c_int),
    }
    for name, (argt, rest) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = argt
        fn.restype = rest
    _lib = L
    return L


def check(rc: int, what: str = ""):
    if rc == VM_OK:
        return
    msg = lib().vm_last_error().decode(errors="replace")
    if rc == VM_ERR_NODEV:
        raise NoDeviceError(msg)
    if rc in (VM_ERR_ARG, VM_ERR_RANGE):
        raise ValueError(f"{what}: {msg}")
    if rc == VM_ERR_OOM:
        raise MemoryError(f"{what}: {msg}")
    raise NativeError(f"{what}: {msg} (code {rc})")


def device_count() -> int:
    n = ctypes.c_int32(0)
    lib().vm_device_count(ctypes.byref(n))
    return int(n.value)


def make_config(cfg) -> VmConfig:
    c = VmConfig()
    c.voxel_size = float(cfg.voxel_size)
    c.region_dim = int(cfg.region_dim)
    c.hit_delta = math.log(cfg.p_hit / (1.0 - cfg.p_hit))       # occupancy.py:20-35
    c.miss_delta = math.log(cfg.p_miss / (1.0 - cfg.p_miss))
    for name in ("clamp_min", "clamp_max", "max_ray_range", "segment_length", "tsdf_truncation",
                 "tsdf_max_weight", "ndt_sensor_noise", "ndt_reset_threshold",
                 "ndt_miss_likelihood_threshold"):
        setattr(c, name, float(getattr(cfg, name)))
    return c


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


class NativeMap:
    """Owner of one device map handle (vm_map)."""

    def __init__(self, cfg, mask: int, device: int = 0, initial_regions: int = 256):
        self._cfg = make_config(cfg)
        h = ctypes.c_void_p()
        check(lib().vm_map_create(ctypes.byref(self._cfg), mask, device, initial_regions,
                                  ctypes.byref(h)), "vm_map_create")
        self._h = h
        self.device = device

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            lib().vm_map_destroy(h)
            self._h = None

    __del__ = close

    def reset(self):
        check(lib().vm_map_reset(self._h), "vm_map_reset")

    def set_stream(self, stream_handle: int | None):
        check(lib().vm_map_set_stream(self._h, ctypes.c_void_p(stream_handle or 0)),
              "vm_map_set_stream")

    def region_count(self) -> int:
        n = ctypes.c_int64()
        check(lib().vm_map_region_count(self._h, ctypes.byref(n)), "vm_map_region_count")
        return int(n.value)

    def region_keys(self, first: int, count: int) -> np.ndarray:
        out = np.empty(max(count, 1), dtype=np.int64)
        if count:
            check(lib().vm_map_region_keys(self._h, first, count, _ptr(out)), "region_keys")
        return out[:count]

    def ensure_regions(self, packed_keys) -> np.ndarray:
        keys = np.ascontiguousarray(packed_keys, dtype=np.int64)
        slots = np.empty(max(len(keys), 1), dtype=np.int32)
        check(lib().vm_map_ensure_regions(self._h, _ptr(keys), len(keys), _ptr(slots)),
              "ensure_regions")
        return slots[:len(keys)]

    def export_select(self, slots, kind: int, threshold: float = 0.0):
        """(region index into `slots`, local index) of the voxels an exporter keeps."""
        sl = np.ascontiguousarray(slots, dtype=np.int32)
        n = I64_t()
        check(lib().vm_export_select(self._h, _ptr(sl), len(sl), kind, float(threshold),
                                     ctypes.byref(n), None, None, 0), "export_select")
        ridx = np.empty(max(n.value, 1), dtype=np.int32)
        li = np.empty(max(n.value, 1), dtype=np.int32)
        if n.value:
            check(lib().vm_export_select(self._h, _ptr(sl), len(sl), kind, float(threshold),
                                         ctypes.byref(n), _ptr(ridx), _ptr(li), len(ridx)),
                  "export_select")
        return ridx[:n.value], li[:n.value]

    def export_gather(self, layer_id: int, slots, ridx, li, dtype, components: int):
        sl = np.ascontiguousarray(slots, dtype=np.int32)
        out = np.empty((max(len(li), 1), components), dtype=dtype)
        if len(li):
            check(lib().vm_export_gather(self._h, layer_id, _ptr(sl), len(sl), _ptr(ridx),
                                         _ptr(li), len(li), _ptr(out)), "export_gather")
        return out[:len(li)]

    def read_layer(self, slot: int, layer_id: int, out: np.ndarray):
        check(lib().vm_map_read_layer(self._h, slot, layer_id, _ptr(out), out.nbytes),
              "read_layer")

    def write_layer(self, slot: int, layer_id: int, arr: np.ndarray):
        arr = np.ascontiguousarray(arr)
        check(lib().vm_map_write_layer(self._h, slot, layer_id, _ptr(arr), arr.nbytes),
              "write_layer")

    def layer_ptr(self, slot: int, layer_id: int) -> int:
        p = ctypes.c_void_p()
        check(lib().vm_map_layer_ptr(self._h, slot, layer_id, ctypes.byref(p)), "layer_ptr")
        return int(p.value or 0)

    # -- recency and eviction (vm_map_evict_regions) ----------------------
    def set_batch_counter(self, counter: int):
        check(lib().vm_map_set_batch_counter(self._h, int(counter) & 0xFFFFFFFF),
              "vm_map_set_batch_counter")

    def region_last_access(self, first: int, count: int) -> np.ndarray:
        out = np.zeros(max(count, 0), dtype=np.uint32)
        if count > 0:
            check(lib().vm_map_region_last_access(self._h, first, count, _ptr(out)),
                  "vm_map_region_last_access")
        return out

    def set_spill(self, directory: str, layer_ids):
        ids = np.asarray(list(layer_ids), dtype=np.int32)
        check(lib().vm_map_set_spill(self._h, str(directory).encode(), _ptr(ids), len(ids)),
              "vm_map_set_spill")

    def evict_regions(self, packed_keys) -> int:
        keys = np.asarray(list(packed_keys), dtype=np.int64)
        n = ctypes.c_int64()
        check(lib().vm_map_evict_regions(self._h, _ptr(keys), len(keys), ctypes.byref(n)),
              "vm_map_evict_regions")
        return int(n.value)

    def reload_region(self, packed_key: int) -> int:
        slot = ctypes.c_int32()
        check(lib().vm_map_reload_region(self._h, int(packed_key), ctypes.byref(slot)),
              "vm_map_reload_region")
        return int(slot.value)

    def spilled_keys(self) -> list[int]:
        n = ctypes.c_int64()
        check(lib().vm_map_spilled_keys(self._h, None, 0, ctypes.byref(n)), "vm_map_spilled_keys")
        out = np.zeros(max(n.value, 1), dtype=np.int64)
        check(lib().vm_map_spilled_keys(self._h, _ptr(out), n.value, ctypes.byref(n)),
              "vm_map_spilled_keys")
        return [int(x) for x in out[:n.value]]

    # -- region sharding (vm_shard_*; device buffers are passed as ints) --
    def shard_config(self, rank: int, world: int):
        check(lib().vm_shard_config(self._h, rank, world), "vm_shard_config")

    def shard_begin(self, rays: VmRays, mode: str = "occupancy") -> tuple[int, int]:
        """Discover this rank's slice; returns (bound on the requests, #new
        sample voxels): occupancy -- new regions; NDT-OM -- prefetched
        regions (every ghost among them is requested)."""
        counts = (ctypes.c_int64 * 2)()
        check(lib().vm_shard_begin(self._h, ctypes.byref(rays), MODES.index(mode), EXEC_DETERMINISTIC,
                                   ctypes.cast(counts, ctypes.c_void_p)), "vm_shard_begin")
        return int(counts[0]), int(counts[1])

    def shard_ndt_bits(self, req_ptr: int, nreq: int, bits_ptr: int):
        check(lib().vm_shard_ndt_bits(self._h, ctypes.c_void_p(req_ptr), nreq,
                                      ctypes.c_void_p(bits_ptr)), "vm_shard_ndt_bits")

    def shard_ndt_mark(self, keys_ptr: int, bits_ptr: int, n: int):
        check(lib().vm_shard_ndt_mark(self._h, ctypes.c_void_p(keys_ptr), ctypes.c_void_p(bits_ptr),
                                      n), "vm_shard_ndt_mark")

    def shard_lists(self, req_ptr: int, req_cap: int, marks_ptr: int, marks_cap: int,
                    world: int) -> list[int]:
        counts = (ctypes.c_int64 * (1 + world))()
        check(lib().vm_shard_lists(self._h, ctypes.c_void_p(req_ptr), req_cap,
                                   ctypes.c_void_p(marks_ptr), marks_cap,
                                   ctypes.cast(counts, ctypes.c_void_p)), "vm_shard_lists")
        return [int(x) for x in counts]

    def shard_prepare(self, req_ptr: int, nreq: int, marks_ptr: int, nmarks: int):
        check(lib().vm_shard_prepare(self._h, ctypes.c_void_p(req_ptr), nreq,
                                     ctypes.c_void_p(marks_ptr), nmarks), "vm_shard_prepare")

    def shard_walk(self):
        check(lib().vm_shard_walk(self._h), "vm_shard_walk")

    def shard_export(self, out_ptr: int, cap_per: int, world: int):
        counts = (ctypes.c_int64 * world)()
        rc = lib().vm_shard_export(self._h, ctypes.c_void_p(out_ptr), cap_per,
                                   ctypes.cast(counts, ctypes.c_void_p))
        return rc, [int(x) for x in counts]

    def shard_import(self, in_ptr: int, n: int):
        check(lib().vm_shard_import(self._h, ctypes.c_void_p(in_ptr), n), "vm_shard_import")

    def shard_finish(self) -> VmStats:
        st = VmStats()
        check(lib().vm_shard_finish(self._h, ctypes.byref(st)), "vm_shard_finish")
        return st

    def integrate_many(self, rays: list, mode: str, deterministic: bool) -> list:
        """One vm_integrate_many call over a sequence of VmRays batches."""
        n = len(rays)
        arr = (VmRays * max(n, 1))(*rays)
        sts = (VmStats * max(n, 1))()
        check(lib().vm_integrate_many(self._h, arr, n, MODES.index(mode),
                                      EXEC_DETERMINISTIC if deterministic else EXEC_CAS, sts),
              "vm_integrate_many")
        return list(sts)[:n]

    def integrate(self, rays: VmRays, mode: str, deterministic: bool) -> VmStats:
        st = VmStats()
        check(lib().vm_integrate(self._h, ctypes.byref(rays), MODES.index(mode),
                                 EXEC_DETERMINISTIC if deterministic else EXEC_CAS,
                                 ctypes.byref(st)), "vm_integrate")
        return st


def rays_from_records(records: np.ndarray, on_device_ptr: int | None = None) -> VmRays:
    r = VmRays()
    r.format = RAYS_OHMB1
    r.count = len(records) if on_device_ptr is None else int(records)
    if on_device_ptr is None:
        assert records.dtype.itemsize == 40 and records.flags.c_contiguous
        r.records = records.ctypes.data
        r.on_device = 0
    else:
        r.records = on_device_ptr
        r.on_device = 1
    return r


def rays_from_arrays(origins, ends, has_sample, intensity=None) -> tuple[VmRays, tuple]:
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    e = np.ascontiguousarray(ends, dtype=np.float64).reshape(-1, 3)
    h = np.ascontiguousarray(has_sample, dtype=np.uint8).reshape(-1)
    it = None if intensity is None else np.ascontiguousarray(intensity, dtype=np.float32)
    r = VmRays()
    r.format = RAYS_F64
    r.on_device = 0
    r.count = len(o)
    r.origins, r.ends, r.has_sample = o.ctypes.data, e.ctypes.data, h.ctypes.data
    r.intensity = it.ctypes.data if it is not None else None
    return r, (o, e, h, it)  # keep the arrays alive


def walk_voxels_native(ox, oy, oz, ex, ey, ez, cell):
    """_kernels.walk_voxels_native (_kernels.pyx:214-228) on the GPU."""
    cap = 4096
    coords = np.empty((cap, 3), dtype=np.int64)
    t0 = np.empty(cap)
    t1 = np.empty(cap)
    n = ctypes.c_int64()
    rc = lib().vm_walk_voxels(float(ox), float(oy), float(oz), float(ex), float(ey), float(ez),
                              float(cell), cap, _ptr(coords), _ptr(t0), _ptr(t1), ctypes.byref(n))
    if rc == VM_ERR_ARG and n.value > cap:
        raise RuntimeError("walk overflow")
    check(rc, "vm_walk_voxels")
    k = int(n.value)
    return coords[:k].copy(), t0[:k].copy(), t1[:k].copy()


def ndt_hypot(ab) -> np.ndarray:
    """math.hypot over the rows of ab (n x 2) with the NDT fold's device
    restatement (ndt.py:37-52 calls it inside cholupdate3)."""
    ab = np.ascontiguousarray(ab, dtype=np.float64).reshape(-1, 2)
    out = np.empty(len(ab))
    check(lib().vm_ndt_hypot(_ptr(ab), len(ab), _ptr(out)), "vm_ndt_hypot")
    return out


def hash_mix(key: int) -> int:
    """_kernels.hash_mix (_kernels.pyx:127-129)."""
    return int(lib().vm_hash_mix(int(key)))


def kernels_integrate_occupancy(origins, ends, has_sample, n, tkeys, tvals, tsize, occ_ptrs,
                                mean_ptrs, count_ptrs, dhit_ptrs, ddist_ptrs, voxel_size,
                                region_dim, hit_delta, miss_delta, clamp_min, clamp_max,
                                retry_limit, walk_cap, stream=0):
    """_kernels.integrate_occupancy (_kernels.pyx:376-470) on the GPU.

    Every array argument is a DEVICE pointer (int); pass 0 for an absent
    mean/count or decay pointer array, like the reference's empty arrays
    (_kernels.pyx:393-394).  Returns (cas_retries, cas_failures,
    region_misses, visits)."""
    st = (ctypes.c_int64 * 4)()
    P = ctypes.c_void_p
    check(lib().vm_kernels_integrate_occupancy(
        P(origins), P(ends), P(has_sample), int(n), P(tkeys), P(tvals), int(tsize), P(occ_ptrs),
        P(mean_ptrs or 0), P(count_ptrs or 0), P(dhit_ptrs or 0), P(ddist_ptrs or 0),
        float(voxel_size), int(region_dim), float(hit_delta), float(miss_delta),
        float(clamp_min), float(clamp_max), int(retry_limit), int(walk_cap),
        ctypes.cast(st, P), P(stream or 0)), "vm_kernels_integrate_occupancy")
    return tuple(int(x) for x in st)


def shard_owner(packed_key: int, world: int) -> int:
    """Owner rank of a region in a `world`-way sharded map (vm_shard_owner)."""
    return int(lib().vm_shard_owner(int(packed_key), int(world)))


def probe_red_rate(device: int = 0, footprint_bytes: int = 64 << 20, reps: int = 5) -> float:
    """Measured L2 atomic (RED.ADD u32, random addresses) throughput, /s: the
    ceiling of the walk's per-visit update (vm_probe_red_rate)."""
    out = ctypes.c_double()
    check(lib().vm_probe_red_rate(device, footprint_bytes, reps, ctypes.byref(out)),
          "vm_probe_red_rate")
    return out.value

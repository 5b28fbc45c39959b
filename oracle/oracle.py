"""ctypes view of the C oracle (vm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product
package.  It is the checker the CUDA path is compared against.

The oracle restates voxmap's *sequential* executor
(/root/reference/pkg/src/voxmap/engine.py:213-237, reference.py:35-186).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libvm_oracle.so"

MODES = ("occupancy", "decay", "ndt-om", "ndt-tm", "tsdf", "counts")

# layers.py:22-31  (name -> (id, dtype, components))
LAYERS = {
    "occupancy": (1, np.float32, 1),
    "mean": (2, np.uint32, 1),
    "mean_count": (3, np.uint32, 1),
    "cov_sqrt": (4, np.float32, 6),
    "hit_count": (5, np.uint32, 1),
    "miss_count": (6, np.uint32, 1),
    "intensity": (7, np.float32, 2),
    "decay_hits": (8, np.uint32, 1),
    "decay_distance": (9, np.float64, 1),
    "tsdf": (10, np.float32, 2),
}
MODE_LAYERS = {
    "occupancy": ("occupancy", "mean", "mean_count"),
    "decay": ("occupancy", "mean", "mean_count", "decay_hits", "decay_distance"),
    "ndt-om": ("occupancy", "mean", "mean_count", "cov_sqrt"),
    "ndt-tm": ("occupancy", "mean", "mean_count", "cov_sqrt", "hit_count", "miss_count",
               "intensity"),
    "tsdf": ("tsdf",),
    # checker aid: per-voxel hit / miss visits of the occupancy walk
    "counts": ("hit_count", "miss_count"),
}
STAT_NAMES = ("rays_in", "rays_processed", "segments", "voxel_visits", "cas_retries",
              "cas_failures", "region_misses", "regions_touched")


class OrcConfig(ctypes.Structure):
    _fields_ = [
        ("voxel_size", ctypes.c_double),
        ("region_dim", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("hit_delta", ctypes.c_double),
        ("miss_delta", ctypes.c_double),
        ("clamp_min", ctypes.c_double),
        ("clamp_max", ctypes.c_double),
        ("max_ray_range", ctypes.c_double),
        ("segment_length", ctypes.c_double),
        ("tsdf_truncation", ctypes.c_double),
        ("tsdf_max_weight", ctypes.c_double),
        ("ndt_sensor_noise", ctypes.c_double),
        ("ndt_reset_threshold", ctypes.c_double),
        ("ndt_miss_likelihood_threshold", ctypes.c_double),
    ]


def build(force: bool = False) -> Path:
    src = HERE / "vm_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        L.orc_map_create.restype = P
        L.orc_map_create.argtypes = [ctypes.POINTER(OrcConfig), ctypes.c_uint32]
        L.orc_map_destroy.argtypes = [P]
        L.orc_map_region_count.restype = ctypes.c_int64
        L.orc_map_region_count.argtypes = [P]
        L.orc_map_regions.restype = ctypes.c_int64
        L.orc_map_regions.argtypes = [P, P, ctypes.c_int64]
        L.orc_map_layer.restype = P
        L.orc_map_layer.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int32]
        L.orc_map_layer_create.restype = P
        L.orc_map_layer_create.argtypes = L.orc_map_layer.argtypes
        L.orc_integrate.restype = ctypes.c_int
        L.orc_integrate.argtypes = [P, P, P, P, P, ctypes.c_int64, ctypes.c_int32, P]
        L.orc_walk.restype = ctypes.c_int64
        L.orc_walk.argtypes = [ctypes.c_double] * 7 + [P, P, P, ctypes.c_int64]
        L.orc_preprocess.restype = ctypes.c_int64
        L.orc_preprocess.argtypes = [ctypes.POINTER(OrcConfig), P, P, P, ctypes.c_int64,
                                     ctypes.c_int32, P, P, P, P, ctypes.c_int64, P]
        L.orc_prefetch_regions.restype = ctypes.c_int64
        L.orc_prefetch_regions.argtypes = [ctypes.POINTER(OrcConfig), P, P, P, ctypes.c_int64,
                                           ctypes.c_double, P, ctypes.c_int64]
        L.orc_norm3.restype = ctypes.c_double
        L.orc_norm3.argtypes = [ctypes.c_double] * 3
        L.orc_py_hypot.restype = ctypes.c_double
        L.orc_py_hypot.argtypes = [ctypes.c_double] * 2
        L.orc_hash_mix.restype = ctypes.c_uint64
        L.orc_hash_mix.argtypes = [ctypes.c_int64]
        _lib = L
    return _lib


def make_config(cfg=None, **kw) -> OrcConfig:
    """Build the C config from any MapConfig-like object (attribute names of
    /root/reference/pkg/src/voxmap/config.py:8-28) or keyword overrides."""
    d = dict(voxel_size=0.1, region_dim=32, p_hit=0.7, p_miss=0.4, clamp_min=-2.0,
             clamp_max=3.5, max_ray_range=20.0, segment_length=10.0, tsdf_truncation=0.3,
             tsdf_max_weight=100.0, ndt_sensor_noise=0.05, ndt_reset_threshold=-1.0,
             ndt_miss_likelihood_threshold=0.2)
    if cfg is not None:
        for k in d:
            d[k] = getattr(cfg, k)
    d.update(kw)
    c = OrcConfig()
    for k in ("voxel_size", "clamp_min", "clamp_max", "max_ray_range", "segment_length",
              "tsdf_truncation", "tsdf_max_weight", "ndt_sensor_noise",
              "ndt_reset_threshold", "ndt_miss_likelihood_threshold"):
        setattr(c, k, float(d[k]))
    c.region_dim = int(d["region_dim"])
    # occupancy.py:20-35 (prob_to_logodds)
    c.hit_delta = math.log(d["p_hit"] / (1.0 - d["p_hit"]))
    c.miss_delta = math.log(d["p_miss"] / (1.0 - d["p_miss"]))
    return c


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


class OracleMap:
    """Sequential CPU map: the C oracle's VoxelMap + sequential_reference."""

    def __init__(self, cfg=None, layer_names=("occupancy", "mean", "mean_count"), **kw):
        self.ccfg = make_config(cfg, **kw)
        self.layer_names = tuple(layer_names)
        mask = 0
        for n in self.layer_names:
            mask |= 1 << LAYERS[n][0]
        self.region_dim = self.ccfg.region_dim
        self._h = lib().orc_map_create(ctypes.byref(self.ccfg), mask)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_map_destroy(h)
            self._h = None

    def integrate(self, origins, ends, has_sample, intensity=None, mode="occupancy"):
        o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        e = np.ascontiguousarray(ends, dtype=np.float64).reshape(-1, 3)
        h = np.ascontiguousarray(has_sample, dtype=np.uint8).reshape(-1)
        it = None
        if intensity is not None:
            it = np.ascontiguousarray(intensity, dtype=np.float32).reshape(-1)
        stats = np.zeros(8, dtype=np.int64)
        rc = lib().orc_integrate(self._h, _ptr(o), _ptr(e), _ptr(h), _ptr(it), len(o),
                                 MODES.index(mode), _ptr(stats))
        if rc != 0:
            raise RuntimeError(f"oracle integrate failed ({rc})")
        return dict(zip(STAT_NAMES, (int(x) for x in stats)))

    def integrate_records(self, records, mode="occupancy"):
        """OHMB1 records (rayset.py:19-27) -> f64 rays exactly like
        to_ray_samples (rayset.py:74-84)."""
        o = records["origin"].astype(np.float64)
        e = records["end"].astype(np.float64)
        h = (records["flags"] & 1).astype(np.uint8)
        return self.integrate(o, e, h, records["intensity"].astype(np.float32), mode)

    def region_keys(self):
        n = lib().orc_map_region_count(self._h)
        out = np.zeros((max(n, 1), 3), dtype=np.int64)
        lib().orc_map_regions(self._h, _ptr(out), n)
        return [tuple(int(c) for c in row) for row in out[:n]]

    def layer(self, rk, name):
        lid, dt, comp = LAYERS[name]
        p = lib().orc_map_layer(self._h, int(rk[0]), int(rk[1]), int(rk[2]), lid)
        if not p:
            return None
        n = self.region_dim ** 3 * comp
        buf = (ctypes.c_char * (n * np.dtype(dt).itemsize)).from_address(p)
        return np.frombuffer(buf, dtype=dt, count=n).copy()

    def set_layer(self, rk, name, values):
        lid, dt, comp = LAYERS[name]
        p = lib().orc_map_layer_create(self._h, int(rk[0]), int(rk[1]), int(rk[2]), lid)
        n = self.region_dim ** 3 * comp
        arr = np.ascontiguousarray(values, dtype=dt).reshape(-1)
        assert arr.size == n
        ctypes.memmove(p, arr.ctypes.data, arr.nbytes)


def walk(origin, end, cell):
    """traversal._walk_grid (traversal.py:52-111)."""
    o = [float(c) for c in origin]
    e = [float(c) for c in end]
    cap = sum(abs(math.floor(e[a] / cell) - math.floor(o[a] / cell)) for a in range(3)) + 2
    coords = np.zeros((cap, 3), dtype=np.int64)
    t0 = np.zeros(cap)
    t1 = np.zeros(cap)
    n = lib().orc_walk(*o, *e, float(cell), _ptr(coords), _ptr(t0), _ptr(t1), cap)
    if n < 0:
        raise RuntimeError("walk overflow")
    return coords[:n].copy(), t0[:n].copy(), t1[:n].copy()


def preprocess(origins, ends, has_sample, segment=True, cfg=None, **kw):
    """engine._preprocess: returns (seg_origins, seg_ends, seg_has, seg_ray, processed)."""
    c = make_config(cfg, **kw)
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    e = np.ascontiguousarray(ends, dtype=np.float64).reshape(-1, 3)
    h = np.ascontiguousarray(has_sample, dtype=np.uint8).reshape(-1)
    cap = 8 * len(o) + 8
    so = np.zeros((cap, 3))
    se = np.zeros((cap, 3))
    sh = np.zeros(cap, dtype=np.uint8)
    sr = np.zeros(cap, dtype=np.int64)
    processed = np.zeros(1, dtype=np.int64)
    n = lib().orc_preprocess(ctypes.byref(c), _ptr(o), _ptr(e), _ptr(h), len(o),
                             1 if segment else 0, _ptr(so), _ptr(se), _ptr(sh), _ptr(sr), cap,
                             _ptr(processed))
    if n < 0:
        raise RuntimeError("preprocess overflow")
    return so[:n], se[:n], sh[:n], sr[:n], int(processed[0])


def prefetch_regions(seg_o, seg_e, seg_has, extra=0.0, cfg=None, **kw):
    """engine.prefetch_regions: distinct region coords touched by the segments."""
    c = make_config(cfg, **kw)
    so = np.ascontiguousarray(seg_o, dtype=np.float64)
    se = np.ascontiguousarray(seg_e, dtype=np.float64)
    sh = np.ascontiguousarray(seg_has, dtype=np.uint8)
    cap = 64 * len(so) + 1024
    out = np.zeros((cap, 3), dtype=np.int64)
    k = lib().orc_prefetch_regions(ctypes.byref(c), _ptr(so), _ptr(se), _ptr(sh), len(so),
                                   float(extra), _ptr(out), cap)
    if k < 0:
        raise RuntimeError("prefetch overflow")
    return out[:k]


def norm3(x, y, z):
    return lib().orc_norm3(float(x), float(y), float(z))


def py_hypot(a, b):
    return lib().orc_py_hypot(float(a), float(b))


def hash_mix(key):
    return int(lib().orc_hash_mix(int(key)))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1

"""Region-hashed voxel store whose payload lives in HBM.

Mirror of voxmap.store (store.py:28-225) for the ray-integration path.
The authoritative copy of every layer is the device region pool owned by
the CUDA runtime (csrc/vm_runtime.cu); `Region.buffers[name]` hands out a
host mirror (numpy array) fetched lazily from the device.  Mirrors that the
caller modified are written back before the next batch, so host writes
(`set_voxel_values`, `region.buffers[..][:] = ...`) behave as in the
reference.  Mirrors handed out before a batch are stale after it: access
`region.buffers[name]` again (the reference's own tests always do).
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import _native
from . import layers as layermod
from .config import MapConfig
from .keys import VoxelKey, key_for_point, local_index, pack_region_coord, unpack_region_coord

MAP_MAGIC = b"OHMR1"


class _Buffers:
    """Mapping layer name -> host mirror of one region's device buffer."""

    __slots__ = ("_region",)

    def __init__(self, region):
        self._region = region

    def __getitem__(self, name):
        return self._region._vmap._mirror(self._region, name)

    def __contains__(self, name):
        return name in self._region._vmap.layer_names

    def __iter__(self):
        return iter(self._region._vmap.layer_names)

    def __len__(self):
        return len(self._region._vmap.layer_names)

    def keys(self):
        return self._region._vmap.layer_names

    def items(self):
        return [(n, self[n]) for n in self]

    def values(self):
        return [self[n] for n in self]


class Region:
    """One dense block of voxels (store.py:28-39), backed by a device slot."""

    __slots__ = ("key", "slot", "_vmap")

    def __init__(self, key, slot: int, vmap):
        self.key = key
        self.slot = slot
        self._vmap = vmap

    @property
    def last_access(self) -> int:
        """The last batch whose prefetch reached the region (the device
        stamps it, engine.py:99-118) or host access (get_region)."""
        return self._vmap._last_access(self)

    @last_access.setter
    def last_access(self, value: int):
        self._vmap._host_touch[self.key] = int(value)

    @property
    def buffers(self) -> _Buffers:
        return _Buffers(self)


class VoxelMap:
    """Layered sparse voxel map in HBM with O(1) region-hash addressing."""

    def __init__(self, cfg: MapConfig, layer_names=("occupancy", "mean", "mean_count"),
                 spill_dir=None, device: int = 0, initial_regions: int = 256):
        self.cfg = cfg
        self.layers = layermod.resolve(layer_names)
        self._regions: dict[tuple[int, int, int], Region] = {}
        self.batch_counter = 0
        self._spill_dir = Path(spill_dir) if spill_dir is not None else None
        self._native = _native.NativeMap(cfg, layermod.layer_mask(layer_names), device,
                                         initial_regions)
        if self._spill_dir is not None:
            self._native.set_spill(str(self._spill_dir), [s.layer_id for s in self.layers])
        self._known = 0          # device slots mirrored into self._regions
        self._mirrors = {}       # (slot, name) -> (array, pristine copy)
        self._host_touch = {}    # region key -> batch counter of the last host access
        self._last = None        # device last-access stamps per slot (cached per batch)

    # -- region access --------------------------------------------------

    @property
    def layer_names(self) -> tuple[str, ...]:
        return tuple(s.name for s in self.layers)

    def has_layers(self, names) -> bool:
        return set(names) <= set(self.layer_names)

    @property
    def regions(self) -> dict:
        """region key -> Region (store.py:45-52).  The device owns the regions;
        this host index is built lazily, on first access after the batches
        that created them, so integrating a batch costs no per-region Python
        work."""
        self._sync_regions()
        return self._regions

    @property
    def region_count(self) -> int:
        return int(self._native.region_count())

    def _note_batch(self, regions_total: int):
        """After a batch: the device's last-access stamps changed."""
        self._last = None

    def _begin_batch(self):
        """Before a batch: its Region.last_access stamp (the counter the
        caller just advanced, engine.py:190)."""
        self._native.set_batch_counter(self.batch_counter)
        self._last = None

    def _last_access(self, region: Region) -> int:
        if self._last is None or len(self._last) < self._known:
            self._last = self._native.region_last_access(0, self._known)
        dev = int(self._last[region.slot]) if region.slot < len(self._last) else 0
        return max(dev, self._host_touch.get(region.key, 0))

    def _sync_regions(self):
        """Mirror device-created regions (slot order = creation order)."""
        n = self._native.region_count()
        if n > self._known:
            for i, packed in enumerate(self._native.region_keys(self._known, n - self._known)):
                rk = unpack_region_coord(int(packed))
                self._regions[rk] = Region(rk, self._known + i, self)
            self._known = n
            self._last = None

    def _reindex(self):
        """The device compacted its pool (eviction): rebuild the host index."""
        self._mirrors.clear()
        self._regions = {}
        self._known = 0
        self._last = None
        self._sync_regions()

    def get_region(self, rk, create: bool = False) -> Region | None:
        rk = (int(rk[0]), int(rk[1]), int(rk[2]))
        region = self.regions.get(rk)
        if region is None and (create or rk in self._spilled_set()):
            # ensure_regions reloads a spilled region transparently
            # (store.py:67-77: get_region reloads from the spill file)
            self._native.ensure_regions([pack_region_coord(rk)])
            self._sync_regions()
            region = self.regions.get(rk)
        if region is not None:
            region.last_access = self.batch_counter
        return region

    def _spilled_set(self) -> set:
        return {unpack_region_coord(k) for k in self._native.spilled_keys()}

    def get_or_create_region(self, rk) -> Region:
        return self.get_region(rk, create=True)

    def clear(self):
        """Drop every region (device pool capacity is kept)."""
        self._mirrors.clear()
        self._native.reset()
        self._regions.clear()
        self._host_touch.clear()
        self._known = 0
        self._last = None

    # -- eviction (store.py:112-174; OHMS1 written by the runtime) ----------

    def spill_dir(self) -> Path:
        if self._spill_dir is None:
            raise RuntimeError("map was created without a spill directory")
        self._spill_dir.mkdir(parents=True, exist_ok=True)
        return self._spill_dir

    def evict_stale_regions(self, age: int) -> int:
        """Spill regions not touched within the last `age` batches to disk
        (zlib, lossless; the same OHMS1 files as the reference) and release
        their HBM.  A later batch -- or get_region -- that reaches a spilled
        region reloads it transparently."""
        self.spill_dir()
        self.flush_host_writes()
        cutoff = self.batch_counter - age
        stale = [pack_region_coord(rk) for rk, r in self.regions.items() if r.last_access < cutoff]
        if not stale:
            return 0
        evicted = self._native.evict_regions(stale)
        if evicted:
            self._reindex()
        return evicted

    def _reload_all_spilled(self) -> None:
        for packed in sorted(self._native.spilled_keys()):
            self._native.reload_region(packed)
        self._sync_regions()

    # -- host mirrors ---------------------------------------------------

    def _mirror(self, region: Region, name: str) -> np.ndarray:
        key = (region.slot, name)
        hit = self._mirrors.get(key)
        if hit is not None:
            return hit[0]
        spec = layermod.BY_NAME[name]
        if name not in self.layer_names:
            raise KeyError(name)
        arr = np.empty(self.cfg.voxels_per_region * spec.components, dtype=spec.dtype)
        self._native.read_layer(region.slot, spec.layer_id, arr)
        self._mirrors[key] = (arr, arr.copy())
        return arr

    def flush_host_writes(self):
        """Write modified host mirrors back to HBM and drop all mirrors."""
        for (slot, name), (arr, pristine) in self._mirrors.items():
            if not np.array_equal(arr.view(np.uint8), pristine.view(np.uint8)):
                self._native.write_layer(slot, layermod.BY_NAME[name].layer_id, arr)
        self._mirrors.clear()

    # -- voxel access (store.py:84-110) ---------------------------------

    def voxel_values(self, layer_name: str, key: VoxelKey):
        region = self.get_region(key.region)
        if region is None:
            return None
        spec = layermod.BY_NAME[layer_name]
        idx = local_index(key.local, self.cfg.region_dim)
        buf = region.buffers[layer_name]
        if spec.components == 1:
            return buf[idx]
        return buf[idx * spec.components:(idx + 1) * spec.components]

    def set_voxel_values(self, layer_name: str, key: VoxelKey, values) -> None:
        region = self.get_or_create_region(key.region)
        spec = layermod.BY_NAME[layer_name]
        idx = local_index(key.local, self.cfg.region_dim)
        buf = region.buffers[layer_name]
        if spec.components == 1:
            buf[idx] = values
        else:
            buf[idx * spec.components:(idx + 1) * spec.components] = values

    def voxel_values_at(self, layer_name: str, point):
        return self.voxel_values(layer_name, key_for_point(point, self.cfg))

    # -- persistence (store.py:178-225, OHMR1; device -> host sync) -------

    def save(self, path) -> None:
        self._reload_all_spilled()
        with open(path, "wb") as fh:
            fh.write(MAP_MAGIC)
            fh.write(struct.pack("<d I I", self.cfg.voxel_size, self.cfg.region_dim,
                                 len(self.layers)))
            for spec in self.layers:
                fh.write(struct.pack("<I", spec.layer_id))
            fh.write(struct.pack("<Q", len(self.regions)))
            for rk in sorted(self.regions):
                fh.write(struct.pack("<3q", *rk))
                for spec in self.layers:
                    fh.write(self.regions[rk].buffers[spec.name].tobytes())

    @classmethod
    def load(cls, path, cfg: MapConfig | None = None, spill_dir=None, device: int = 0):
        raw = Path(path).read_bytes()
        if raw[:5] != MAP_MAGIC:
            raise ValueError(f"{path} is not a voxel map file")
        off = 5
        voxel_size, region_dim, nlayers = struct.unpack_from("<d I I", raw, off)
        off += 16
        ids = struct.unpack_from(f"<{nlayers}I", raw, off)
        off += 4 * nlayers
        names = tuple(layermod.BY_ID[i].name for i in ids)
        if cfg is None:
            cfg = MapConfig(voxel_size=voxel_size, region_dim=region_dim)
        elif cfg.voxel_size != voxel_size or cfg.region_dim != region_dim:
            raise ValueError("config does not match file geometry")
        (nregions,) = struct.unpack_from("<Q", raw, off)
        off += 8
        vmap = cls(cfg, names, spill_dir=spill_dir, device=device,
                   initial_regions=max(64, int(nregions)))
        for _ in range(nregions):
            rk = struct.unpack_from("<3q", raw, off)
            off += 24
            region = vmap.get_or_create_region(rk)
            for spec in vmap.layers:
                n = cfg.voxels_per_region * spec.components * spec.dtype.itemsize
                vmap._native.write_layer(region.slot, spec.layer_id,
                                         np.frombuffer(raw[off:off + n], dtype=spec.dtype))
                off += n
        return vmap

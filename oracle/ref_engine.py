"""CPU reference arm, end to end: the reference package's own engine.

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py cpu_baseline / cpu_sweep).
Imports the UNMODIFIED reference package `voxmap` 0.1.0 from baseline/_ref
(installed there by `pip install --no-deps --target baseline/_ref <copy of
/root/reference/pkg>`; git-ignored, it travels to the GPU box with the
snapshot) and times `voxmap.submit_batch(vmap, rays, mode,
ExecutorOptions(worker_count=W))` exactly as a user calls it: Python clip /
segment / prefetch, the native kernel on W threads, and -- for NDT -- the
Python phase 2 (engine.py:175-210, 266-302).  The figure is the reference's
own `BatchStats.rays_per_second` (wall_time excludes `to_ray_samples`,
engine.py:191,209), best of `repeats`.
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF_PKG = ROOT / "baseline" / "_ref"


def load_voxmap():
    """The installed reference package, or None when it is absent."""
    if not (REF_PKG / "voxmap" / "__init__.py").exists():
        return None
    if str(REF_PKG) not in sys.path:
        sys.path.insert(0, str(REF_PKG))
    try:
        import voxmap  # noqa: F401
        from voxmap import layers  # noqa: F401
    except Exception:  # pragma: no cover - broken install
        return None
    return sys.modules["voxmap"]


def time_submit_batch(cfg_kw: dict, mode: str, warm_batches, timed_batch, workers: int,
                      repeats: int = 1):
    """rays/s of the reference engine on `timed_batch` (OHMB1 records) after
    the untimed `warm_batches` built the map state it lands on."""
    vx = load_voxmap()
    if vx is None:
        return None
    from voxmap.layers import MODE_LAYERS
    best = 0.0
    for _ in range(max(1, repeats)):
        vm = vx.VoxelMap(vx.MapConfig(**cfg_kw), MODE_LAYERS[mode])
        opts = vx.ExecutorOptions(worker_count=workers)
        for rec in warm_batches:
            vx.submit_batch(vm, vx.to_ray_samples(rec), mode, opts)
        rays = vx.to_ray_samples(timed_batch)
        st = vx.submit_batch(vm, rays, mode, opts)
        best = max(best, st.rays_per_second)
    return best

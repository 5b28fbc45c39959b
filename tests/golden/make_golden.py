"""Generate golden vectors by running the REFERENCE itself (voxmap 0.1.0).

Usage (in the build container, where /root/reference exists):

    python tests/golden/make_golden.py [--ref-src /tmp/refpkg/src]

If --ref-src is not given the reference package is copied from
/root/reference/pkg to /tmp/voxmap_refpkg and its Cython extension is
built there (the reference's own setup.py, unmodified).  Nothing from the
reference is copied into this repository: only the *outputs* (ray inputs,
stats, region key sets and per-layer SHA-256 digests, plus walk / norm /
hypot vectors) are written to tests/golden/*.npz.

The fixtures pin:
  * traversal._walk_grid visit sequences        (traversal.py:52-111)
  * RaySample.length / clip / segment            (traversal.py:40-42,140-178)
  * math.hypot as used by ndt.cholupdate3        (ndt.py:42)
  * sequential_reference end states per mode     (engine.py:213-237)
"""
from __future__ import annotations

import argparse
import hashlib
import math
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def ensure_ref(src: str | None) -> Path:
    if src:
        return Path(src)
    dst = Path("/tmp/voxmap_refpkg")
    if not (dst / "src" / "voxmap").exists():
        shutil.copytree("/root/reference/pkg", dst)
    if not list((dst / "src" / "voxmap").glob("_kernels*.so")):
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=dst,
                       check=True, capture_output=True)
    return dst / "src"


def layer_digest(vmap, name) -> str:
    h = hashlib.sha256()
    for rk in sorted(vmap.regions):
        h.update(np.asarray(rk, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(vmap.regions[rk].buffers[name]).tobytes())
    return h.hexdigest()


def random_records(n, spread, seed, max_len=35.0):
    from voxmap.rayset import records_from_arrays
    r = np.random.default_rng(seed)
    o = r.uniform(-spread, spread, (n, 3))
    d = r.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    L = r.uniform(0.01, max_len, n)
    return records_from_arrays(np.arange(n) * 1e-6, o, o + d * L[:, None],
                               r.uniform(5, 50, n), r.random(n) < 0.8)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-src", default=None)
    args = ap.parse_args()
    sys.path.insert(0, str(ensure_ref(args.ref_src)))
    import voxmap
    from voxmap import (MapConfig, SceneSpec, VoxelMap, generate_scene, sequential_reference,
                        to_ray_samples)
    from voxmap.layers import MODE_LAYERS
    from voxmap.traversal import RaySample, clip_ray, segment_ray, walk_voxels_global

    assert voxmap.__version__ == "0.1.0"
    rng = np.random.default_rng(2024)

    # -- walk vectors (test_kernels.py:14-27, test_traversal.py:18-50) ------
    pts = rng.uniform(-8.0, 8.0, (700, 6))
    # exact-grid and corner inputs (tie-breaks, zero components, -0.0)
    grid = rng.integers(-40, 40, (600, 6)) * 0.05
    pts = np.concatenate([pts, grid, [[0.05, 0.05, 0.05, 0.15, 0.15, 0.15],
                                      [0.05, 0.05, 0.05, 0.15, 0.15, 0.05],
                                      [0.05, 0.05, 0.05, -0.25, 0.05, 0.05],
                                      [-0.0, 0.0, -0.0, 0.3, -0.0, 0.0],
                                      [0.05, 0.05, 0.05, 0.05, 0.05, 0.05]]])
    off, coords, t0s, t1s = [0], [], [], []
    for p in pts:
        c, a, b = walk_voxels_global(p[:3], p[3:], MapConfig())
        coords.append(c.reshape(-1, 3))
        t0s.append(a)
        t1s.append(b)
        off.append(off[-1] + len(a))
    np.savez_compressed(HERE / "walk.npz", pts=pts, offsets=np.array(off),
                        coords=np.concatenate(coords).astype(np.int32), t0=np.concatenate(t0s),
                        t1=np.concatenate(t1s), cell=0.1)

    # -- norm / hypot / clip+segment vectors --------------------------------
    v = rng.uniform(-30, 30, (4000, 3)) * 10.0 ** rng.uniform(-3, 0, (4000, 1))
    norms = np.array([float(np.linalg.norm(x)) for x in v])
    hy = np.concatenate([rng.normal(size=(4000, 2)) * 10.0 ** rng.integers(-300, 300, (4000, 2)),
                         rng.normal(size=(4000, 2))])
    hyp = np.array([math.hypot(a, b) for a, b in hy])
    rec = random_records(3000, 30.0, 11, max_len=45.0)
    so, se, sh, sr = [], [], [], []
    for i, ray in enumerate(to_ray_samples(rec)):
        if ray.length == 0.0:
            continue
        for s in segment_ray(clip_ray(ray, MapConfig()), MapConfig()):
            so.append(s.origin)
            se.append(s.end)
            sh.append(s.has_sample)
            sr.append(i)
    np.savez_compressed(HERE / "arith.npz", v=v, norms=norms, hy=hy, hyp=hyp, seg_records=rec,
                        seg_o=np.array(so), seg_e=np.array(se), seg_has=np.array(sh, np.uint8),
                        seg_ray=np.array(sr))

    # -- end-to-end sequential_reference cases ------------------------------
    cases = []

    def add(name, cfgkw, batches, modes):
        cfg = MapConfig(**cfgkw)
        for mode in modes:
            vm = VoxelMap(cfg, MODE_LAYERS[mode])
            stats = []
            for b in batches:
                s = sequential_reference(vm, to_ray_samples(b), mode)
                stats.append([s.rays_in, s.rays_processed, s.segments, s.voxel_visits,
                              s.cas_retries, s.cas_failures, s.region_misses, s.regions_touched])
            cases.append(dict(name=f"{name}/{mode}", cfg=cfgkw, mode=mode,
                              batches=[np.asarray(b) for b in batches], stats=np.array(stats),
                              regions=np.array(sorted(vm.regions), dtype=np.int64).reshape(-1, 3),
                              digests={n: layer_digest(vm, n) for n in MODE_LAYERS[mode]}))
            print(f"{name}/{mode}: {len(vm.regions)} regions, visits {stats[-1][3]}", flush=True)

    all_modes = ("occupancy", "decay", "ndt-om", "ndt-tm", "tsdf")
    corr = generate_scene(SceneSpec(kind="corridor", rate=20000, duration=0.05, seed=1))
    add("corridor", {}, [corr], all_modes)
    of = generate_scene(SceneSpec(kind="open-field", rate=20000, duration=0.06, seed=2,
                                  noise=0.01))
    add("open-field", {}, [of], all_modes)
    poles = generate_scene(SceneSpec(kind="thin-poles", rate=20000, duration=0.1, seed=7,
                                     noise=0.005))
    add("thin-poles-x2", {}, [poles[:1000], poles[1000:], poles[:1000], poles[1000:]], all_modes)
    add("random", {}, [random_records(800, 30.0, 21), random_records(800, 30.0, 22)], all_modes)
    add("random-05-r16", dict(voxel_size=0.05, region_dim=16),
        [random_records(500, 5.0, 31)] * 2, ("occupancy", "decay", "ndt-tm", "tsdf"))
    add("random-odd", dict(voxel_size=0.25, region_dim=7, max_ray_range=30.0,
                           segment_length=4.0),
        [random_records(400, 5.0, 41)] * 2, ("occupancy", "ndt-om", "tsdf"))

    out = {}
    for i, c in enumerate(cases):
        p = f"c{i}_"
        out[p + "name"] = np.array(c["name"])
        out[p + "mode"] = np.array(c["mode"])
        out[p + "cfg"] = np.array(repr(c["cfg"]))
        out[p + "nbatches"] = np.array(len(c["batches"]))
        for j, b in enumerate(c["batches"]):
            out[p + f"b{j}"] = b
        out[p + "stats"] = c["stats"]
        out[p + "regions"] = c["regions"]
        for n, d in c["digests"].items():
            out[p + "digest_" + n] = np.array(d)
    out["ncases"] = np.array(len(cases))
    np.savez_compressed(HERE / "scenes.npz", **out)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()

"""Golden exporter outputs from the REFERENCE itself (voxmap 0.1.0).

Usage (build container, where /root/reference exists):

    python tests/golden/make_exports.py [--ref-src /tmp/voxmap_refpkg/src]

For every sequential_reference case of scenes.npz (make_golden.py), the
reference re-integrates the same batches and writes each export format that
applies to the mode with its own exporters (exporters.py:14-159).  Only the
outputs -- the exported files, compressed -- are stored in exports.npz.
"""
from __future__ import annotations

import argparse
import ast
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import ensure_ref  # noqa: E402

FORMATS = {
    "occupancy": ("occupied-ply",),
    "decay": ("occupied-ply", "decay-csv"),
    "ndt-om": ("occupied-ply", "ndt-csv"),
    "ndt-tm": ("occupied-ply", "ndt-csv"),
    "tsdf": ("tsdf-csv",),
}


HEAD_ROWS = 20000


def exact_digest(text: bytes, ncols: int) -> str:
    """sha256 over the first `ncols` columns of every data row (the columns
    that must match exactly: voxel center and integer counts)."""
    import hashlib
    h = hashlib.sha256()
    for line in text.decode().splitlines()[1:]:
        h.update((",".join(line.split(",")[:ncols]) + "\n").encode())
    return h.hexdigest()


def store(out: dict, k: int, case: int, fmt: str, n: int, text: bytes):
    """Full text for small files; for long CSVs the header + first HEAD_ROWS
    rows in full and a digest of the exact columns of all rows."""
    out[f"e{k}_case"] = np.array(case)
    out[f"e{k}_fmt"] = np.array(fmt)
    out[f"e{k}_count"] = np.array(n)
    lines = text.split(b"\n")
    if fmt.endswith("-csv") and len(lines) > HEAD_ROWS + 2:
        out[f"e{k}_text"] = np.frombuffer(b"\n".join(lines[:HEAD_ROWS + 1]) + b"\n", dtype=np.uint8)
        out[f"e{k}_exact4"] = np.array(exact_digest(text, 4))
        out[f"e{k}_partial"] = np.array(1)
    else:
        out[f"e{k}_text"] = np.frombuffer(text, dtype=np.uint8)
        out[f"e{k}_partial"] = np.array(0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-src", default=None)
    args = ap.parse_args()
    sys.path.insert(0, str(ensure_ref(args.ref_src)))
    from voxmap import MapConfig, VoxelMap, sequential_reference, to_ray_samples
    from voxmap.exporters import export_map
    from voxmap.layers import MODE_LAYERS

    z = np.load(HERE / "scenes.npz", allow_pickle=False)
    out = {}
    k = 0
    for i in range(int(z["ncases"])):
        p = f"c{i}_"
        mode = str(z[p + "mode"])
        cfgkw = ast.literal_eval(str(z[p + "cfg"]))
        vm = VoxelMap(MapConfig(**cfgkw), MODE_LAYERS[mode])
        for j in range(int(z[p + "nbatches"])):
            sequential_reference(vm, to_ray_samples(z[p + f"b{j}"]), mode)
        for fmt in FORMATS[mode]:
            with tempfile.NamedTemporaryFile(suffix=".txt") as f:
                n = export_map(vm, fmt, f.name)
                text = Path(f.name).read_bytes()
            store(out, k, i, fmt, n, text)
            print(str(z[p + "name"]), fmt, n, len(text), flush=True)
            k += 1
    out["nexports"] = np.array(k)
    np.savez_compressed(HERE / "exports.npz", **out)


if __name__ == "__main__":
    main()

"""GPU exporters against the reference's own exporter output (exporters.py:14-159).

tests/golden/exports.npz holds the files the reference wrote for every
sequential_reference case of scenes.npz (make_exports.py).  The device map is
built from the same batches on the deterministic path and exported here:

* occupied-ply and tsdf-csv: byte-identical (occupancy, mean, mean_count and
  tsdf are bit-exact on this path);
* ndt-csv and decay-csv: same rows in the same order, integer columns exact,
  real columns within the reference's own executor tolerances
  (test_engine.py:52-63) carried through the printed precision.
"""
import ast
import io

import numpy as np
import pytest

from tests._util import GOLDEN

pytestmark = pytest.mark.gpu

from paper_2206_06079_b200 import ExecutorOptions, MapConfig, VoxelMap, submit_batch  # noqa: E402
from paper_2206_06079_b200.exporters import export_map  # noqa: E402
from paper_2206_06079_b200.layers import MODE_LAYERS  # noqa: E402

Z = np.load(GOLDEN / "exports.npz", allow_pickle=False)
S = np.load(GOLDEN / "scenes.npz", allow_pickle=False)
EXPORTS = [(int(Z[f"e{k}_case"]), str(Z[f"e{k}_fmt"]), k) for k in range(int(Z["nexports"]))]
_maps = {}


def _map(case):
    if case not in _maps:
        _maps.clear()  # one device map at a time (cases are grouped)
        p = f"c{case}_"
        mode = str(S[p + "mode"])
        vm = VoxelMap(MapConfig(**ast.literal_eval(str(S[p + "cfg"]))), MODE_LAYERS[mode])
        for j in range(int(S[p + "nbatches"])):
            submit_batch(vm, S[p + f"b{j}"], mode, ExecutorOptions(deterministic=True))
        _maps[case] = vm
    return _maps[case]


def _rows(text):
    lines = text.decode().splitlines()
    return lines[0], [ln.split(",") for ln in lines[1:]]


@pytest.mark.parametrize("case,fmt,k", EXPORTS,
                         ids=[f"{S[f'c{c}_name']}-{f}" for c, f, _ in EXPORTS])
def test_export_matches_reference(case, fmt, k, tmp_path):
    vm = _map(case)
    path = tmp_path / "out.txt"
    n = export_map(vm, fmt, path)
    want = Z[f"e{k}_text"].tobytes()
    got = path.read_bytes()
    assert n == int(Z[f"e{k}_count"])
    if fmt in ("occupied-ply", "tsdf-csv"):
        assert got == want
        return
    h1, r1 = _rows(got)
    h2, r2 = _rows(want)
    if int(Z[f"e{k}_partial"]):
        # long CSV: exact columns (center, hits) of every row by digest, the
        # first rows in full below
        from tests.golden.make_exports import exact_digest
        assert exact_digest(got, 4) == str(Z[f"e{k}_exact4"])
        r1 = r1[:len(r2)]
    assert h1 == h2 and len(r1) == len(r2)
    ints = {"ndt-csv": (3, 14, 15), "decay-csv": (3,)}[fmt]
    for a, b in zip(r1, r2):
        assert a[:3] == b[:3]  # voxel center: same voxel, same order
        for j in range(3, len(a)):
            if j in ints or a[j] == "" or b[j] == "":
                assert a[j] == b[j], (j, a, b)
            else:
                assert float(a[j]) == pytest.approx(float(b[j]), rel=1e-4, abs=2e-5), (j, a, b)

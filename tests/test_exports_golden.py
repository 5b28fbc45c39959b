"""CPU checks of the exporter fixtures (tests/golden/exports.npz, written by
the reference's own exporters, exporters.py:44-159, via make_exports.py):
every stored file is well-formed and its row count matches the count the
reference returned."""
import numpy as np

from tests._util import GOLDEN

HEADER = {"occupied-ply": 7, "ndt-csv": 1, "tsdf-csv": 1, "decay-csv": 1}


def test_export_fixtures_consistent():
    z = np.load(GOLDEN / "exports.npz", allow_pickle=False)
    n = int(z["nexports"])
    assert n >= 30
    fmts = set()
    for k in range(n):
        fmt = str(z[f"e{k}_fmt"])
        fmts.add(fmt)
        text = z[f"e{k}_text"].tobytes().decode()
        lines = text.splitlines()
        count = int(z[f"e{k}_count"])
        if fmt == "occupied-ply":
            assert lines[2] == f"element vertex {count}"
        if int(z[f"e{k}_partial"]):
            assert len(lines) - HEADER[fmt] < count
            assert len(str(z[f"e{k}_exact4"])) == 64
        else:
            assert len(lines) - HEADER[fmt] == count
    assert fmts == set(HEADER)

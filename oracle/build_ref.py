"""Compile the reference's own native kernel into oracle/_ref/ (checker only).

The reference's only native code is the Cython module
/root/reference/pkg/src/voxmap/_kernels.pyx (built by pkg/setup.py:5-13 with
`-O3 -std=c11`).  This recipe cythonizes it from where it lies (output C
goes to a temp dir, never into the repo) and links oracle/_ref/_kernels*.so
with the same flags.  The resulting .so is git-ignored but travels to the
GPU box with gpurun, where bench.py --impl reference times it on the host
cores (kernel-only, `_kernels.integrate_occupancy` over pre-built segment
arrays and region table, exactly as engine._run_parallel drives it,
engine.py:240-262).

Nothing here runs when /root/reference is absent (the GPU box): the
prebuilt .so is used as is.
"""
from __future__ import annotations

import shutil
import subprocess
import sys
import sysconfig
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref"
PYX = Path("/root/reference/pkg/src/voxmap/_kernels.pyx")


def built_path() -> Path | None:
    hits = sorted(OUT.glob("_kernels*.so"))
    return hits[0] if hits else None


def build(force: bool = False) -> Path | None:
    if not PYX.exists():
        return built_path()
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    target = OUT / f"_kernels{suffix}"
    if target.exists() and not force and target.stat().st_mtime >= PYX.stat().st_mtime:
        return target
    import numpy
    OUT.mkdir(parents=True, exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        c_file = Path(td) / "_kernels.c"
        subprocess.run([sys.executable, "-m", "cython", "-3", "--module-name", "_kernels",
                        "-o", str(c_file), str(PYX)], check=True, capture_output=True)
        inc = [sysconfig.get_paths()["include"], numpy.get_include()]
        cc = shutil.which("gcc") or "cc"
        cmd = [cc, "-shared", "-fPIC", "-O3", "-std=c11",
               "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION"]
        cmd += [f"-I{p}" for p in inc] + [str(c_file), "-o", str(target), "-lpthread", "-lm"]
        subprocess.run(cmd, check=True, capture_output=True)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))

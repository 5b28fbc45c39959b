"""Build the CUDA extension in-tree: paper_2206_06079_b200/_lib/libvoxmap_b200.so.

One translation unit (csrc/vm_runtime.cu includes the kernels), compiled
for sm_100a only, with -fmad=false so every floating-point operation rounds
exactly like the reference's numpy / CPython arithmetic (see
csrc/vm_device.cuh).  cudart is linked statically so the .so only needs the
driver on the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libvoxmap_b200.so"
INCLUDE = PKG.parent / "include"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart=static",
]


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [INCLUDE / "voxmap_b200.h"]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in sources())


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, f"-I{INCLUDE}", "-o", str(tmp), str(CSRC / "vm_runtime.cu"), "-lz"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        errs = "\n".join(l for l in res.stderr.splitlines()
                          if "error" in l or "warning" in l) or res.stderr[-4000:]
        raise RuntimeError(f"nvcc failed:\n{errs[-6000:]}")
    if verbose:
        print(res.stderr, file=sys.stderr)
    os.replace(tmp, LIB)
    return LIB


def build_variant(name: str, defines: list[str]) -> Path:
    """Dev experiments: the same library built with extra -D flags into
    _lib/<name> (selected at run time with VOXMAP_B200_LIB=<name>)."""
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    out = LIB_DIR / name
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], f"-I{INCLUDE}", "-o", str(out),
           str(CSRC / "vm_runtime.cu"), "-lz"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stderr[-6000:]}")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

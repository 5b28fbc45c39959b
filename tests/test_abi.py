"""CPU-side checks of the C-ABI library and the host mirror of the reference
interface: every function include/voxmap_b200.h declares is exported, the
struct layouts ctypes uses match the header, and without a GPU the product
path fails loudly instead of falling back to the CPU."""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2206_06079_b200 import (ConfigurationError, ExecutorOptions, MapConfig, _native,
                                   read_rayset, records_from_arrays, write_rayset)

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "voxmap_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(vm_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 15, names
    lib = _native.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_100a" in _native.lib().vm_build_info().decode()


def _struct_size(name):
    """sizeof(struct) as the header defines it, via the C compiler."""
    src = f'#include "{HEADER}"\n#include <stdio.h>\nint main(void){{printf("%zu", sizeof({name}));}}\n'
    exe = Path("/tmp") / f"vm_sizeof_{name}"
    subprocess.run(["gcc", "-x", "c", "-", "-o", str(exe)], input=src, text=True, check=True)
    return int(subprocess.run([str(exe)], capture_output=True, text=True).stdout)


@pytest.mark.parametrize("cname,py", [("vm_config", _native.VmConfig), ("vm_stats", _native.VmStats),
                                      ("vm_rays", _native.VmRays)])
def test_ctypes_layouts_match_header(cname, py):
    assert ctypes.sizeof(py) == _struct_size(cname)


def test_hash_mix_needs_no_device():
    # _kernels.hash_mix (_kernels.pyx:105-110,127-129), splitmix64 finalizer
    def ref(k):
        m = (1 << 64) - 1
        h = (k + 0x9E3779B97F4A7C15) & m
        h = ((h ^ (h >> 30)) * 0xBF58476D1CE4E5B9) & m
        h = ((h ^ (h >> 27)) * 0x94D049BB133111EB) & m
        return h ^ (h >> 31)
    for k in (0, 1, 7, 123456789, 2 ** 62 + 5):
        assert _native.hash_mix(k) == ref(k)


@pytest.mark.skipif(_native.device_count() > 0, reason="a GPU is present")
def test_no_device_fails_loudly():
    from paper_2206_06079_b200 import VoxelMap
    with pytest.raises(_native.NoDeviceError):
        VoxelMap(MapConfig())
    with pytest.raises(_native.NativeError):
        _native.walk_voxels_native(0.05, 0.05, 0.05, 0.35, 0.15, 0.05, 0.1)


def test_executor_options_errors_match_reference():
    # engine.py:67-79
    with pytest.raises(ValueError):
        ExecutorOptions(worker_count=0)
    with pytest.raises(ValueError):
        ExecutorOptions(kind="gpu")
    with pytest.raises(ValueError):
        ExecutorOptions(worker_count=2, kind="sequential")
    assert ExecutorOptions().use_deterministic
    assert not ExecutorOptions(worker_count=4).use_deterministic
    assert issubclass(ConfigurationError, Exception)


def test_mapconfig_validation():
    with pytest.raises(ValueError):
        MapConfig(voxel_size=0.0)
    with pytest.raises(ValueError):
        MapConfig(p_hit=0.4)
    assert MapConfig().region_size == pytest.approx(3.2)


def test_ohmb1_round_trip(tmp_path):
    r = np.random.default_rng(0)
    n = 100
    rec = records_from_arrays(np.arange(n) * 1e-3, r.normal(size=(n, 3)), r.normal(size=(n, 3)),
                              r.uniform(5, 50, n), r.random(n) < 0.5)
    p = tmp_path / "x.ohmb"
    write_rayset(p, rec)
    back = read_rayset(p)
    assert back.dtype.itemsize == 40
    assert np.array_equal(back.view(np.uint8), rec.view(np.uint8))

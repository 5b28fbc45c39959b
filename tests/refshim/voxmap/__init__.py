"""`voxmap` alias package -- TEST INFRASTRUCTURE ONLY.

Maps the reference package's import paths (voxmap, voxmap.engine,
voxmap._kernels, ...) onto paper_2206_06079_b200, so the reference's own test
files (/root/reference/pkg/tests, installed unmodified beside the reference
package in baseline/_ref/ref_tests) run against the GPU path
(tests/test_gpu_reference_suite.py).  The only reference code it loads is
the synthetic scene generator scenes.py -- test input, not the hot path --
from the installed reference package.
"""
import importlib.util
import sys
from pathlib import Path

from paper_2206_06079_b200 import *  # noqa: F401,F403  (the drop-in surface)
from paper_2206_06079_b200 import __all__ as _ours  # noqa: F401

_REF = Path(__file__).resolve().parents[3] / "baseline" / "_ref" / "voxmap" / "scenes.py"


def _load_scenes():
    spec = importlib.util.spec_from_file_location("voxmap.scenes", _REF)
    mod = importlib.util.module_from_spec(spec)
    sys.modules["voxmap.scenes"] = mod
    spec.loader.exec_module(mod)
    return mod


scenes = _load_scenes()
SCENE_KINDS, SceneSpec, generate_scene = scenes.SCENE_KINDS, scenes.SceneSpec, scenes.generate_scene

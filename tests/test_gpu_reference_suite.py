"""The reference's own test files, unmodified, against the GPU path.

baseline/_ref holds the reference package (pip-installed, unmodified) and its
test suite (pkg/tests); tests/refshim/voxmap aliases the reference's import
paths onto paper_2206_06079_b200 (the drop-in claim: a user of voxmap
switches by changing the import).  Selected: the engine, traversal and
native-kernel suites, the store / keys / occupancy / sub-voxel / ray-set
units, and the acceptance criteria that are about results (01-04, 07-10);
05 / 06 / 11 time the reference's thread pool and its online drop rate
under overload, which the GPU path does not reproduce (it does not fall
behind).  Skipped where baseline/_ref is absent."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
REF_TESTS = ROOT / "baseline" / "_ref" / "ref_tests"
RUNNER = ROOT / "tests" / "refshim" / "run_reference_tests.py"

SUITES = {
    "engine": ["test_engine.py"],
    "traversal_kernels": ["test_traversal.py", "test_kernels.py"],
    "units": ["test_store.py", "test_keys.py", "test_occupancy.py", "test_subvoxel.py",
              "test_rayset.py"],
    "acceptance": ["test_acceptance.py", "-k",
                   "test_01 or test_02 or test_03 or test_04 or test_07 or test_08 or "
                   "test_09 or test_10"],
}


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference test suite not installed in baseline/_ref")
@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suite_passes(suite):
    res = subprocess.run([sys.executable, str(RUNNER), "-q", "-x", *SUITES[suite]],
                         capture_output=True, text=True, timeout=1800)
    tail = "\n".join(res.stdout.splitlines()[-15:])
    print(tail)
    assert res.returncode == 0, tail + res.stderr[-2000:]

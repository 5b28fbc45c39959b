"""Run reference test files against the GPU path through the `voxmap`
alias package.  usage: python tests/refshim/run_reference_tests.py
<pytest args...> (paths under baseline/_ref/ref_tests).  Test infrastructure."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]

if __name__ == "__main__":
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "refshim"), str(ROOT),
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "--rootdir",
           str(ROOT / "baseline" / "_ref" / "ref_tests"), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=env, cwd=str(ROOT / "baseline" / "_ref" / "ref_tests")))

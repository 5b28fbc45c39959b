import gc
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the checker (C oracle) is built; the CUDA library is built by
    __graft_entry__.build() (the GPU tests fail loudly without it)."""
    from oracle import oracle
    oracle.build()


@pytest.fixture(autouse=True)
def _release_device_maps():
    """VoxelMap <-> Region reference cycles keep device maps (HBM pools) alive
    until the cyclic GC runs; collect after every test so a long GPU session
    does not accumulate them."""
    yield
    gc.collect()

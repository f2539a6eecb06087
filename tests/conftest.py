import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def dev():
    """The device C-ABI, initialised on GPU 0. GPU tests fail loudly when the
    native library is missing (no fallback)."""
    import paper_1307_2100_b200 as T
    lib = T.native.device()
    T.check(lib.tcb_init(0), "tcb_init")
    return lib

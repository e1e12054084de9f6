import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLD = ROOT / "tests" / "golden"
REF_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and libpsb200.so (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


@pytest.fixture(scope="session")
def gold():
    import numpy as np

    def load(name):
        return np.load(GOLD / name, allow_pickle=False)
    return load


@pytest.fixture(scope="session")
def reference_pkg():
    """The read-only reference package (build container only)."""
    if not REF_SRC.exists():
        pytest.skip("reference package not present (GPU box)")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import pseudospec
    return pseudospec


@pytest.fixture(scope="session")
def gpu():
    """Library handle on cuda:0; on a GPU box a missing library is a failure, not a skip."""
    from paper_2605_04550_b200 import _lib
    return _lib.handle(0)


@pytest.fixture(scope="session")
def refpkg_any():
    """The unmodified reference package from baseline/_ref (travels to the GPU box) or the
    read-only checkout; skip when neither exists."""
    for cand in (ROOT / "baseline" / "_ref", REF_SRC):
        if (cand / "pseudospec").exists():
            if str(cand) not in sys.path:
                sys.path.insert(0, str(cand))
            import pseudospec
            return pseudospec
    pytest.skip("reference package not available")

"""Shared fixtures.  `gpu` tests need a B200 and the built libigs_b200.so;
everything else runs on the CPU (oracle pinning, host logic, ABI exports)."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def port():
    import oracle
    if not oracle.available("port"):
        oracle.build()
    return oracle.get("port")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference library (oracle/_ref); skipped when absent."""
    import oracle
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return oracle.get("reference")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
    return load


@pytest.fixture(scope="session")
def gctx():
    """One device context for the gpu tests (fails loudly without the .so)."""
    from paper_2407_01866_b200 import Context
    ctx = Context(0)
    yield ctx
    ctx.close()

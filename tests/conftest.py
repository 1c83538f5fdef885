import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build (if stale) the product library and the oracles once per session.
    On the GPU box the prebuilt files are used (no /root/reference there)."""
    from paper_1510_05218_b200 import _build
    try:
        _build.build()
    except Exception:
        if not os.path.exists(_build.LIB):
            raise
    from oracle import oracle
    if not os.path.exists(oracle.C_LIB):
        oracle.build()
    yield

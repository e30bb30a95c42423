import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def port():
    from oracle.pyoracle import Port

    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle

    if not pyoracle.ref_available():
        try:
            pyoracle.build_ref()
        except Exception:
            pass
    if not pyoracle.ref_available():
        pytest.skip("compiled reference (oracle/_ref) not available on this machine")
    return pyoracle.Ref()

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun); parity tests through the C ABI")


@pytest.fixture(scope="session")
def orc():
    from oracle_bind import load_oracle
    return load_oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_bind import load_ref
    lib = load_ref()
    if lib is None:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return lib


@pytest.fixture(scope="session")
def prb():
    """The product C-ABI library (loads only; no GPU needed to load)."""
    from paper_2112_05923_b200 import _lib
    return _lib.lib()

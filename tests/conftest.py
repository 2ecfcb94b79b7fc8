"""Shared fixtures.  `gpu` marks tests that need a B200; everything else runs
on the CPU-only build box.  The checkers (oracle/) are test infrastructure."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle
    return pyoracle.load_c()


@pytest.fixture(scope="session")
def ref():
    """The reference library itself (oracle/_ref), or skip when it was not built."""
    from oracle import pyoracle
    r = pyoracle.load_ref()
    if r is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return r


@pytest.fixture(scope="session")
def pd():
    import paper_2008_01938_b200 as pd
    pd.lib()
    return pd


@pytest.fixture(scope="session")
def gpu(pd):
    if pd.device_count() < 1:
        pytest.fail("no sm_100 GPU visible for a gpu-marked test")
    return pd

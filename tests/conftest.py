import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle pin")


@pytest.fixture(scope="session")
def built_lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2307_08606_b200 import _lib
    return _lib.lib()

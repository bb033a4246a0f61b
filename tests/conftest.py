import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")


@pytest.fixture(scope="session", autouse=True)
def _built_c_libs():
    import __graft_entry__ as ge
    ge.build_oracle()
    ge.build_synth()
    yield

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (B200) and the built libpk_b200.so")


import pytest  # noqa: E402


@pytest.fixture
def plan():
    """set_plan_options(**fields) for the test (packtrain_b200.h pk_plan_options:
    pins the MLP path's kernel families); the previous plan is restored after."""
    from paper_2002_02885_b200 import _lib
    prev = _lib.plan_options()
    yield _lib.set_plan_options
    _lib.set_plan_options(**prev)

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle and the product library once (no-op when up to date)."""
    import subprocess
    subprocess.check_call(["make", "-s", "-C", ROOT, "all"], stdout=subprocess.DEVNULL)

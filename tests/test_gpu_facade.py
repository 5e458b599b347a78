"""The reference-shaped C++ facade (include/steinmcl_b200.hpp) drives the B200
engine end to end (examples/facade_demo.cpp, built by `make`)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_facade_builds():
    assert os.path.exists(os.path.join(ROOT, "examples", "facade_demo"))


@pytest.mark.gpu
def test_facade_demo_runs():
    out = subprocess.run([os.path.join(ROOT, "examples", "facade_demo")], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("facade_demo ok"), out.stdout

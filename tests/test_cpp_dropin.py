"""Runs the C++ drop-in test driver (tests/cpp/test_dropin.cpp): the
reference's own test cases against include/ddsg_b200.hpp."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
DRIVER = ROOT / "build" / "test_dropin"


def _driver():
    if not DRIVER.exists():
        import sys

        sys.path.insert(0, str(ROOT))
        import __graft_entry__

        __graft_entry__._load_builder().build_library()
    return DRIVER


def test_dropin_cpu_cases():
    r = subprocess.run([str(_driver()), "cpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


@pytest.mark.gpu
def test_dropin_gpu_cases():
    r = subprocess.run([str(_driver()), "gpu"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout

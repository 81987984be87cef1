"""Runs the C++ drop-in test drivers:
  * tests/cpp/test_dropin.cpp (build/test_dropin): the reference's own test
    cases against include/ddsg_b200.hpp;
  * tests/cpp/test_ref_dropin.cpp (oracle/_ref/test_ref_dropin, built by
    `make -C oracle dropin` where the reference exists and shipped prebuilt):
    the reference headers in place beside the shim -- decompose, INTEGRATION.md's
    to_b200() verbatim, compiled_evaluator with only the namespace changed,
    a reference-written policy.json through the C-ABI -- bit for bit."""
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


REF_DRIVER = ROOT / "oracle" / "_ref" / "test_ref_dropin"


@pytest.mark.gpu
def test_reference_headers_beside_the_shim():
    if not REF_DRIVER.exists():
        pytest.fail(f"{REF_DRIVER} missing: build it with `make -C oracle dropin` (needs /root/reference)")
    r = subprocess.run([str(REF_DRIVER)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout and "0 of 3000 points differ" in r.stdout, r.stdout

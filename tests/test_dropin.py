"""The C++ drop-in layer (include/lamfast, liblamfast.so): a program written
against the reference's lamfast API (tests/cpp/test_dropin.cpp) built and run
against the B200 edition."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_dropin")


@pytest.fixture(scope="module")
def dropin_binary():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1905_05417_b200", "csrc")],
                   check=True, capture_output=True)
    assert os.path.exists(BIN)
    return BIN


def test_dropin_host_side(dropin_binary):
    r = subprocess.run([dropin_binary, "--host-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_dropin_reference_test_cases_on_gpu(dropin_binary):
    r = subprocess.run([dropin_binary], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout

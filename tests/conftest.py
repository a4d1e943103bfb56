import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.checkers import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.checkers import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def gpu():
    import paper_1905_05417_b200 as lf
    lib = lf.library()  # fails loudly when the CUDA library is missing
    if lib.lf_device_count() < 1:
        pytest.fail("GPU test on a host without a usable CUDA device")
    return lf


def assert_csr_match(got, want, rtol=1e-12):
    """Pattern bit-exact; values within rtol * max|K_want| (BASELINE.json)."""
    rp, cols, vals = got
    rp0, cols0, vals0 = want
    assert np.array_equal(np.asarray(rp), np.asarray(rp0)), "row offsets differ"
    assert np.array_equal(np.asarray(cols), np.asarray(cols0)), "column indices differ"
    scale = float(np.abs(vals0).max()) if len(vals0) else 0.0
    err = float(np.abs(np.asarray(vals) - np.asarray(vals0)).max()) if len(vals0) else 0.0
    assert err <= rtol * scale, f"max |dK| = {err:.3e} > {rtol:g} * {scale:.3e}"
    return err / scale if scale else 0.0

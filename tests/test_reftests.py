"""The reference's OWN unit suites, compiled unmodified against the drop-in.

tests/cpp/build_reftests.sh compiles /root/reference/proj/tests/{unit_main,
test_splines, test_quadrature, test_geometry, test_materials, test_sparse,
test_assembly, test_fast, test_voigt_free}.cpp -- the reference's unit_tests
target minus test_bench.cpp (sweep harness, out of scope) -- against
include/lamfast (the drop-in headers), liblamfast.so + liblamfast_b200.so and
a from-scratch doctest subset (tests/cpp/doctest_subset/doctest.h), into
build/reftests/unit_tests.  On the B200 every test case must pass; on a host
without a GPU the host-side cases pass and every device case fails loudly
with the library's "no CUDA device available" error (no CPU fallback).
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "reftests", "unit_tests")
N_CASES = 79  # TEST_CASEs in the eight suites


def _run():
    if not os.path.exists(BIN):
        pytest.skip("build/reftests/unit_tests not built (needs /root/reference at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=1800)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", p.stdout)
    assert m, p.stdout[-2000:] + p.stderr[-2000:]
    return p, int(m.group(1)), int(m.group(2)), int(m.group(3))


def test_reference_unit_suites_host_cases_pass_and_device_cases_fail_loudly():
    import paper_1905_05417_b200 as lf
    if lf.library().lf_device_count() > 0:
        pytest.skip("a GPU is present: the -m gpu test runs the suites")
    p, total, passed, failed = _run()
    assert total == N_CASES
    assert passed >= 50, p.stdout[-3000:]
    # every failing assertion is the library refusing to run without a device
    blocks = re.split(r"\n(?=\S+:\d+: ERROR)", p.stdout)
    for b in blocks:
        if ": ERROR" in b:
            assert "no CUDA device available" in b, b[:1000]


@pytest.mark.gpu
def test_reference_unit_suites_pass_on_the_b200():
    p, total, passed, failed = _run()
    assert p.returncode == 0 and failed == 0, p.stdout[-6000:]
    assert total == passed == N_CASES

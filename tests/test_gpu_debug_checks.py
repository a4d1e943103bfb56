"""Bounds-checked device build (make debug -> build/dbg, LF_CHECK traps on any
out-of-range device write; the stand-in for compute-sanitizer, which the GPU
pool does not allow).  Runs every kernel family on small cases through it, in
a subprocess so a trap cannot poison this process's CUDA context."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DBG = os.path.join(ROOT, "build", "dbg", "liblamfast_b200.so")


def test_all_kernel_families_pass_bounds_checks(gpu):
    if not os.path.exists(DBG):
        pytest.skip("bounds-checked library not built (make -C paper_1905_05417_b200/csrc debug)")
    env = dict(os.environ, LAMFAST_LIB=DBG)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "LF_CHECK failed" not in r.stdout + r.stderr, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.strip().startswith("ok")

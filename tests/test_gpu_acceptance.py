"""The reference's acceptance suite (acceptance.cpp) restated on the GPU, at
its full grid -- device fast vs device standard vs device Voigt-free -- plus
its timing gates and the determinism tests of test_assembly.cpp:229-240 /
test_fast.cpp:427-439.  Device verification kernels (lf_csr_*) compute the
norms, so the grid runs without host-side sparse algebra."""
import time

import numpy as np
import pytest

from oracle.checkers import csr_rel_diff
from paper_1905_05417_b200 import problem as P

pytestmark = pytest.mark.gpu


def _angles(kind, m, p):
    if kind == 0:
        return [0.0 if l % 2 == 0 else 0.5 * P.PI for l in range(m)]
    if kind == 1:
        return [[0.0, 0.25 * P.PI, -0.25 * P.PI, 0.5 * P.PI][l % 4] for l in range(m)]
    rng = P.MT19937(7 + m + p)
    return [(rng() / 2 ** 32 - 0.5) * P.PI for _ in range(m)]


def _translation_residual(k):
    """||K t||_inf / ||K||_F over the three rigid translations (acceptance.cpp:95-104)."""
    import scipy.sparse as sp
    n = len(k.row_ptr) - 1
    a = sp.csr_matrix((k.values, k.cols, k.row_ptr), shape=(n, n))
    worst = 0.0
    for d in range(3):
        t = np.zeros(n)
        t[d::3] = 1.0
        worst = max(worst, np.abs(a @ t).max())
    return worst / np.sqrt((k.values ** 2).sum())


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("elems", [1, 2, 4])
def test_acceptance_equivalence_grid(gpu, p, elems):
    """acceptance.cpp:58-123: p in 1..4 x elements in {1,2,4} x m in
    {1,2,3,8,32} x 3 layups: standard vs fast vs Voigt-free <= 1e-12, rigid
    translations annihilated <= 1e-12, K symmetric."""
    for m in (1, 2, 3, 8, 32):
        for kind in (0, 1, 2):
            prob = P.cube_problem(p, elems, 1, _angles(kind, m, p))
            std = gpu.assemble_standard(prob)
            fast = gpu.assemble_fast(prob)
            vf = gpu.assemble_voigt_free(prob)
            assert fast.nnz == std.nnz == vf.nnz
            assert np.array_equal(fast.cols, std.cols)
            assert csr_rel_diff(fast.astuple(), std.astuple()) <= 1e-12, (p, elems, m, kind)
            assert csr_rel_diff(vf.astuple(), std.astuple()) <= 1e-12, (p, elems, m, kind)
            assert _translation_residual(fast) <= 1e-12
            assert _translation_residual(std) <= 1e-12


def test_determinism_bitwise(gpu):
    """Repeated assemblies are bit-identical (no atomics anywhere: coloured or
    owner-computes accumulation), for every backend and geometry kind."""
    probs = [P.baseline_config("C2"), P.cube_problem(3, 3, 2, [0.0, 0.7, -0.2], geometry="skewed")]
    for prob in probs:
        for backend in ("fast", "standard", "voigt_free"):
            a = gpu.assemble_with(backend, prob)
            b = gpu.assemble_with(backend, prob)
            assert np.array_equal(a.values, b.values), backend


def test_slabs_are_bitwise_rows_of_the_full_matrix(gpu):
    """A row slab computes exactly the full matrix's rows (same arithmetic per
    value), for any partition -- the multi-GPU result equals the 1-GPU one."""
    import torch
    prob = P.baseline_config("C2")
    full = gpu.assemble_fast(prob)
    for parts in (2, 5):
        got = []
        for part in range(parts):
            b = gpu.slab_bounds(prob, parts, part)
            plan = gpu.Plan(prob, "fast", 0, b["t_begin"], b["t_end"])
            vals = torch.empty(max(1, plan.nnz), dtype=torch.float64, device="cuda")
            plan.assemble(vals.data_ptr())
            plan.synchronize()
            got.append(vals.cpu().numpy()[:plan.nnz])
            plan.close()
        assert np.array_equal(np.concatenate(got), full.values)


def _device_ms(gpu, prob, backend, reps=5):
    import torch
    plan = gpu.Plan(prob, backend, 0)
    vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        plan.assemble(vals.data_ptr())
        plan.synchronize()
        t.append(time.perf_counter() - t0)
    plan.close()
    return float(np.median(t)) * 1e3


def test_acceptance_timing_gates(gpu):
    """acceptance.cpp:127-185 on the device: fast >= 10x standard at p=4, 8x8,
    m=64; fast cost independent of the ply count (max/min <= 2 from m=8 to
    m=64 with one thickness element) while standard grows (>= 4x)."""
    big = P.cube_problem(4, 8, 1, _angles(0, 64, 4))
    t_fast, t_std = _device_ms(gpu, big, "fast"), _device_ms(gpu, big, "standard")
    assert t_std / t_fast >= 10.0, (t_fast, t_std)
    f8 = _device_ms(gpu, P.cube_problem(3, 4, 1, _angles(0, 8, 3)), "fast")
    f64 = _device_ms(gpu, P.cube_problem(3, 4, 1, _angles(0, 64, 3)), "fast")
    s8 = _device_ms(gpu, P.cube_problem(3, 4, 1, _angles(0, 8, 3)), "standard")
    s64 = _device_ms(gpu, P.cube_problem(3, 4, 1, _angles(0, 64, 3)), "standard")
    assert max(f8, f64) / min(f8, f64) <= 2.0, (f8, f64)
    assert s64 / s8 >= 4.0, (s8, s64)

"""Row slabs cut inside thickness rows (function ranges) and the chunked
one-shot pipeline (lf_assemble / lf_assemble_range / lf_assemble_stream).

A function is f = i_t * n_s + i_s (rows 3f .. 3f+2).  A plan or one-shot
call over [f0, f1) must return exactly rows [3 f0, 3 f1) of the full matrix:
the pattern bit-exact (row offsets rebased) and the values bitwise equal to
the full assembly's (the same kernels compute the same entries), and the
oracle's rows within 1e-12 * max|K|."""
import numpy as np
import pytest

from conftest import assert_csr_match
from paper_1905_05417_b200 import problem as P

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def _rows(full, f0, f1):
    rp, cols, vals = full
    z0, z1 = rp[3 * f0], rp[3 * f1]
    return rp[3 * f0:3 * f1 + 1] - z0, cols[z0:z1], vals[z0:z1]


def _oracle_rows(oracle, prob, backend, f0, f1):
    """The oracle's rows of functions [f0, f1), cut from its thickness rows."""
    ns = prob.n_s
    t0, t1 = f0 // ns, -(-f1 // ns)
    rp, cols, vals = oracle.assemble(prob, backend, t0, t1)
    return _rows((rp, cols, vals), f0 - t0 * ns, f1 - t0 * ns)


def _device_range(gpu, prob, backend, f0, f1):
    import torch
    plan = gpu.Plan(prob, backend, 0, f_begin=f0, f_end=f1)
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(max(1, plan.nnz), dtype=torch.int32, device="cuda")
    vals = torch.empty(max(1, plan.nnz), dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    info = (plan.rows, plan.nnz, plan.row_begin, plan.nnz_begin)
    plan.close()
    return (rp.cpu().numpy(), cols[:info[1]].cpu().numpy(), vals[:info[1]].cpu().numpy()), info


MIXED = dict(degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3), knots_v=P.uniform_knots(3, 2),
             knots_t=P.c0_knots(2, 3), interfaces=P.equal_interfaces(3),
             layers=[(P.baseline_orthotropic(), 0.0), (P.isotropic(0.5, 0.3), 0.0), (P.baseline_orthotropic(), 0.6)])


@pytest.mark.parametrize("backend", ["fast", "standard", "voigt_free"])
@pytest.mark.parametrize("case", ["C2", "mixed", "skewed"])
def test_function_range_plans_are_rows_of_the_full_matrix(gpu, oracle, backend, case):
    if case == "C2":
        prob = P.baseline_config("C2")
    elif case == "mixed":
        prob = P.LaminateProblem(**MIXED)
    else:
        prob = P.cube_problem(2, 3, 2, [0.0, 0.9, 0.3], geometry="skewed")
    full = gpu.assemble_with(backend, prob).astuple()
    ns, F = prob.n_s, prob.n_s * prob.n_t
    rng = np.random.default_rng(7)
    ranges = [(0, F), (1, F - 1), (ns // 2, ns // 2 + 1), (ns - 1, ns + 1), (ns + 3, 3 * ns - 2), (0, 0),
              (F - 1, F)]
    ranges += [tuple(sorted(rng.integers(0, F + 1, 2))) for _ in range(4)]
    for f0, f1 in ranges:
        got, (rows, nnz, r0, z0) = _device_range(gpu, prob, backend, f0, f1)
        want = _rows(full, f0, f1)
        assert rows == 3 * (f1 - f0) and r0 == 3 * f0 and z0 == full[0][3 * f0]
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
        assert np.array_equal(got[2], want[2]), (f0, f1)  # bitwise: same kernels, same entries
        if f1 > f0 and backend != "voigt_free":
            assert_csr_match(got, _oracle_rows(oracle, prob, backend, f0, f1), RTOL)


@pytest.mark.parametrize("host_cols", ["1", "0"])
def test_function_range_one_shot_and_balanced_bounds(gpu, monkeypatch, host_cols):
    """lf_assemble_range equals the plan's rows, and lf_slab_bounds_functions'
    parts tile the matrix with nnz balanced to within one function; with the
    columns written on the host (default) and copied from the device pattern
    (LAMFAST_HOST_COLS=0)."""
    monkeypatch.setenv("LAMFAST_HOST_COLS", host_cols)
    prob = P.baseline_config("C2")
    full = gpu.assemble_fast(prob).astuple()
    parts = 5
    nnz = []
    prev = 0
    for part in range(parts):
        b = gpu.slab_bounds_functions(prob, parts, part)
        assert b["f_begin"] == prev
        prev = b["f_end"]
        got = gpu.assemble_range(prob, b["f_begin"], b["f_end"]).astuple()
        want = _rows(full, b["f_begin"], b["f_end"])
        for g, w in zip(got, want):
            assert np.array_equal(g, w)
        assert b["nnz_begin"] == full[0][b["row_begin"]] and b["nnz_end"] == full[0][b["row_end"]]
        nnz.append(b["nnz_end"] - b["nnz_begin"])
    assert prev == prob.n_s * prob.n_t
    assert max(nnz) / (sum(nnz) / parts) <= 1.001


@pytest.mark.parametrize("backend", ["fast", "standard"])
@pytest.mark.parametrize("host_cols", ["1", "0"])
def test_streamed_chunks_equal_one_shot(gpu, monkeypatch, backend, host_cols):
    """lf_assemble_stream with small chunks (many chunks, chunk edges inside
    thickness rows) delivers, in row order, exactly the one-shot CSR; the
    pinned and pageable destinations of lf_assemble give the same arrays.
    Columns written by host threads (per chunk into the staging slot for the
    sink) and copied from the device pattern (LAMFAST_HOST_COLS=0); the
    reference CSR comes from the device-pattern path."""
    import torch
    prob = P.baseline_config("C2")
    monkeypatch.setenv("LAMFAST_HOST_COLS", "0")
    want = gpu.assemble_with(backend, prob).astuple()
    monkeypatch.setenv("LAMFAST_HOST_COLS", host_cols)
    got_rp, got_c, got_v = [np.zeros(1, np.int64)], [], []
    seen = {"rows": 0, "nnz": 0, "chunks": 0}

    def sink(row_begin, rows, nnz_begin, rp, cols, vals):
        assert row_begin == seen["rows"] and nnz_begin == seen["nnz"]
        assert rp[0] == 0 and rp[-1] == len(vals)
        got_rp.append(rp[1:] + nnz_begin)
        got_c.append(cols.copy())
        got_v.append(vals.copy())
        seen["rows"] += rows
        seen["nnz"] += len(vals)
        seen["chunks"] += 1
        return 0

    st = gpu.assemble_stream(prob, sink, backend, max_chunk_nnz=1_000_003)
    assert seen["chunks"] >= 30
    got = (np.concatenate(got_rp), np.concatenate(got_c), np.concatenate(got_v))
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    assert st.operator_builds == (0 if backend == "standard" else 2)
    # pinned host arrays (direct D2H) equal the pageable ones (staged)
    dim, nnz = gpu.pattern_size(prob, backend)
    pinned = (torch.empty(dim + 1, dtype=torch.int64, pin_memory=True),
              torch.empty(nnz, dtype=torch.int32, pin_memory=True),
              torch.empty(nnz, dtype=torch.float64, pin_memory=True))
    import ctypes
    from paper_1905_05417_b200 import abi
    c = prob.to_c()
    abi.check(gpu.library().lf_assemble(ctypes.byref(c), abi.BACKENDS[backend], 0, *[t.data_ptr() for t in pinned],
                                        None))
    for g, w in zip(pinned, want):
        assert np.array_equal(g.numpy(), w)


def test_stream_sink_abort_is_reported(gpu):
    prob = P.baseline_config("C2")
    with pytest.raises(gpu.LamfastError) as e:
        gpu.assemble_stream(prob, lambda *a: 1, max_chunk_nnz=1 << 20)
    assert e.value.kind == "runtime_error"


@pytest.mark.slow
@pytest.mark.parametrize("host_cols", ["1", "0"])
def test_c4_one_shot_chunked_into_pageable_host_memory(gpu, monkeypatch, host_cols):
    """Full C4 (1.92e9 nnz, 23 GB: 12 chunks of <= 2 GiB) through lf_assemble
    into pageable numpy arrays (staged through pinned buffers by host
    threads) equals the device-resident plan's CSR bitwise: with the columns
    written by host threads (default) and with the device pattern copied."""
    import torch
    monkeypatch.setenv("LAMFAST_HOST_COLS", host_cols)
    prob = P.baseline_config("C4")
    got = gpu.assemble_fast(prob)
    plan = gpu.Plan(prob, "fast", 0)
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    assert np.array_equal(got.row_ptr, rp.cpu().numpy())
    step = 1 << 28
    for lo in range(0, plan.nnz, step):
        hi = min(plan.nnz, lo + step)
        assert np.array_equal(got.cols[lo:hi], cols[lo:hi].cpu().numpy())
        assert np.array_equal(got.values[lo:hi], vals[lo:hi].cpu().numpy())
    plan.close()
    del rp, cols, vals, got
    torch.cuda.empty_cache()

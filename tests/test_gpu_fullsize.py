"""Full-size BASELINE configs pinned against the oracle (not against another
device path): row slabs of three thickness functions at the bottom, middle
and top of C3, C4 and C5 -- C5 at its full 192 x 192, p = 3, 128-ply size,
where the top slabs sit past 2^32 in the global CSR -- each compared with
the oracle's rows of the same slab (pattern bit-exact, values within
1e-12 * max|K|), and the slabs' global offsets (lf_slab_bounds, the plan's
nnz_begin) against the oracle's global row offsets (fast.cpp:241-258,
sparse.cpp:30-55)."""
import numpy as np
import pytest

from conftest import assert_csr_match
from paper_1905_05417_b200 import problem as P

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RTOL = 1e-12


def _device_slab(gpu, prob, t0, t1):
    import torch
    plan = gpu.Plan(prob, "fast", 0, t0, t1)
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(max(1, plan.nnz), dtype=torch.int32, device="cuda")
    vals = torch.empty(max(1, plan.nnz), dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    out = (rp.cpu().numpy(), cols[:plan.nnz].cpu().numpy(), vals[:plan.nnz].cpu().numpy())
    info = {"nnz_begin": plan.nnz_begin, "row_begin": plan.row_begin, "nnz": plan.nnz}
    plan.close()
    del rp, cols, vals
    torch.cuda.empty_cache()
    return out, info


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_full_size_boundary_slabs_match_oracle(gpu, oracle, name):
    prob = P.baseline_config(name)
    terms = oracle.fast_terms(prob)
    nt = prob.n_t
    for t in (0, nt // 2, nt - 3):
        got, info = _device_slab(gpu, prob, t, t + 3)
        want = terms.slab(t, t + 3)
        assert_csr_match(got, want, RTOL)
        # global placement: the slab's first entry is the oracle's row offset of row 3 n_s t
        assert info["nnz_begin"] == terms.nnz_before(t)
        assert info["row_begin"] == 3 * prob.n_s * t
        assert info["nnz_begin"] + info["nnz"] == terms.nnz_before(t + 3)
    total = terms.nnz_before(nt)
    assert total == P.sizes(prob)["nnz"]
    if name == "C5":
        assert terms.nnz_before(nt - 3) > 2 ** 32  # the top slab's offsets need int64
    # the multi-GPU cuts: every part's global offsets equal the oracle's
    for parts in (2, 8):
        for part in range(parts):
            b = gpu.slab_bounds(prob, parts, part)
            assert b["nnz_begin"] == terms.nnz_before(b["t_begin"])
            assert b["nnz_end"] == terms.nnz_before(b["t_end"])
    terms.close()


def _device_range(gpu, prob, f0, f1):
    import torch
    plan = gpu.Plan(prob, "fast", 0, f_begin=f0, f_end=f1)
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(max(1, plan.nnz), dtype=torch.int32, device="cuda")
    vals = torch.empty(max(1, plan.nnz), dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    out = (rp.cpu().numpy(), cols[:plan.nnz].cpu().numpy(), vals[:plan.nnz].cpu().numpy())
    info = {"nnz_begin": plan.nnz_begin, "row_begin": plan.row_begin, "nnz": plan.nnz}
    plan.close()
    del rp, cols, vals
    torch.cuda.empty_cache()
    return out, info


@pytest.mark.parametrize("parts", [8, 3])
def test_c5_function_range_cuts_match_oracle(gpu, oracle, parts):
    """The multi-GPU cuts of C5 fall inside thickness rows
    (lf_slab_bounds_functions).  Around every cut of the 8- and 3-way splits,
    a function range straddling it (the last 40 functions of one part and the
    first 40 of the next, plus the matrix's first and last 40) is assembled
    as its own plan and equals the oracle's rows (pattern bit-exact, values
    within 1e-12 * max|K|), at global offsets up to 1.69e10 (> 2^32) that
    must equal the oracle's function offsets."""
    prob = P.baseline_config("C5")
    terms = oracle.fast_terms(prob)
    ns, F = prob.n_s, prob.n_s * prob.n_t
    cuts = [gpu.slab_bounds_functions(prob, parts, k)["f_begin"] for k in range(1, parts)]
    windows = [(0, 40), (F - 40, F)] + [(c - 40, c + 40) for c in cuts]
    for f0, f1 in windows:
        got, info = _device_range(gpu, prob, f0, f1)
        assert info["nnz_begin"] == terms.function_offset(f0)
        assert info["nnz_begin"] + info["nnz"] == terms.function_offset(f1)
        assert info["row_begin"] == 3 * f0
        t0, t1 = f0 // ns, (f1 - 1) // ns + 1
        rp, cols, vals = terms.slab(t0, t1)
        a, e = 3 * (f0 - t0 * ns), 3 * (f1 - t0 * ns)
        want = (rp[a:e + 1] - rp[a], cols[rp[a]:rp[e]], vals[rp[a]:rp[e]])
        assert_csr_match(got, want, RTOL)
    assert max(terms.function_offset(c) for c in cuts) > 2 ** 32 or parts == 3
    terms.close()


def test_c3_standard_slab_rows_are_bitwise_rows_of_the_full_matrix(gpu):
    """The standard (K6) two-phase assembly sums each entry per batch of
    thickness spans; batches are aligned to absolute span multiples, so a row
    slab whose rows straddle a batch boundary (C3: 12 spans per 4 GiB batch,
    boundary between spans 11 and 12, i.e. at thickness function 24, shared by
    both) gets bitwise the full matrix's rows."""
    import torch
    prob = P.baseline_config("C3")
    ns = prob.n_s
    full = gpu.Plan(prob, "standard", 0)
    vals = torch.empty(full.nnz, dtype=torch.float64, device="cuda")
    full.assemble(vals.data_ptr())
    full.synchronize()
    for f0, f1 in [(22 * ns + 17, 26 * ns - 5), (0, 3 * ns), (24 * ns, 25 * ns), (23 * ns + 3, 24 * ns + 9)]:
        plan = gpu.Plan(prob, "standard", 0, f_begin=f0, f_end=f1)
        sv = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
        plan.assemble(sv.data_ptr())
        plan.synchronize()
        z0 = plan.nnz_begin
        assert torch.equal(sv, vals[z0:z0 + plan.nnz]), (f0, f1)
        plan.close()
        del sv
    full.close()
    del vals
    torch.cuda.empty_cache()


@pytest.mark.parametrize("case", ["decompose C4", "decompose C4 folded", "16 angles C3", "16 angles C3 slots",
                                  "6 angles C4 slots"])
def test_full_size_coefficient_form_matches_per_term_form_and_oracle(gpu, oracle, monkeypatch, case):
    """The one-pass forms of the combine for many operator terms at full
    BASELINE size -- the coefficient form (default from 8 terms where rows see
    more than 3: C4 with decompose_angles, 10 terms; forced for C3 with 16
    distinct angles) and the slot form (default from 5 terms where every row
    sees <= 3: C3 with 16 distinct angles, C4 with 6), and C4's
    decompose_angles terms folded per ply configuration (the default on affine
    maps: three terms, per-term kernel) -- against the unfolded per-term
    form with its read-modify-write passes (both thresholds at 1000) on the
    device over the whole matrix (same pattern; values within 1e-12 of
    max|K|), and the first, middle and last thickness rows against the
    oracle."""
    import torch
    slots = case.endswith("slots")
    folded = case.endswith("folded")
    if case.startswith("decompose C4"):
        prob = P.baseline_config("C4").replace(decompose_angles=True)
    else:
        base = P.baseline_config(case.split()[2])
        n = int(case.split()[0])
        prob = base.replace(layers=[(P.baseline_orthotropic(), -1.5 + 3.0 * (k % n) / n)
                                    for k in range(len(base.layers))])
    one_pass = {"LAMFAST_SLOTS_MIN_TERMS": "5" if slots else "1000", "LAMFAST_EFORM_MIN_TERMS": "8",
                "LAMFAST_FOLD_DECOMPOSE": "1" if folded else "0"}
    vals = {}
    for mode in ("8", "1000"):
        env = one_pass if mode == "8" else {"LAMFAST_SLOTS_MIN_TERMS": "1000", "LAMFAST_EFORM_MIN_TERMS": "1000",
                                            "LAMFAST_FOLD_DECOMPOSE": "0"}
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        plan = gpu.Plan(prob, "fast", 0)
        v = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
        plan.assemble(v.data_ptr())
        plan.synchronize()
        vals[mode] = v
        nnz = plan.nnz
        plan.close()
    scale = float(vals["1000"].abs().max())
    assert float((vals["8"] - vals["1000"]).abs().max()) <= 1e-12 * scale
    del vals
    torch.cuda.empty_cache()
    for k, v in one_pass.items():
        monkeypatch.setenv(k, v)
    terms = oracle.fast_terms(prob)
    nt = prob.n_t
    for t in (0, nt // 2, nt - 1):
        got, info = _device_slab(gpu, prob, t, t + 1)
        assert_csr_match(got, terms.slab(t, t + 1), RTOL)
        assert info["nnz_begin"] == terms.nnz_before(t)
    assert terms.nnz_before(nt) == nnz
    terms.close()

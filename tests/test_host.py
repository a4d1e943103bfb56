"""Host-side logic of the product library, CPU only (no compute calls):
C-ABI exports, host setup mirrors, closed-form pattern sizes and slabs,
error mapping, problem builders, and the no-fallback guarantee."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_1905_05417_b200 as lf
from paper_1905_05417_b200 import abi
from paper_1905_05417_b200 import problem as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "tests", "golden", "ref_summaries.json")) as f:
    SUMMARY = json.load(f)


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "lamfast_cuda.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(lf_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = lf.library()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert {n for n, _, _ in abi.SIGNATURES} == set(names)
    assert lib.lf_abi_version() == 1
    assert lib.lf_status_name(2) == b"domain_error"


def test_compute_entry_points_fail_loudly_without_gpu():
    lib = lf.library()
    if lib.lf_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(lf.LamfastError) as e:
        lf.assemble_fast(P.baseline_config("C1"))
    assert "no CUDA device" in str(e.value) and e.value.status == abi.LF_ERR_CUDA
    import numpy as np
    out = (np.empty(8, np.int64), np.empty(8, np.int32), np.empty(8))
    with pytest.raises(lf.LamfastError) as e:
        lf.assemble_slab(P.baseline_config("C1"), 0, 1, out=out)
    assert e.value.status == abi.LF_ERR_CUDA
    prob = P.baseline_config("C1")
    with pytest.raises(lf.LamfastError) as e:
        lf.reference_bilinear(prob, np.zeros(prob.dim), np.zeros(prob.dim))
    assert e.value.status == abi.LF_ERR_CUDA


def test_voigt_and_rotation_match_reference_known_answers(oracle):
    lib = lf.library()
    d = (ctypes.c_double * 36)()
    assert lib.lf_voigt_from_constants(ctypes.byref(abi.Orthotropic(*P.pagano())), d) == 0
    np.testing.assert_allclose(np.array(d).reshape(6, 6), SUMMARY["known_answers"]["pagano_D"],
                               atol=1e-14)
    r = (ctypes.c_double * 36)()
    assert lib.lf_rotate_inplane(d, 0.6, r) == 0
    np.testing.assert_allclose(np.array(r).reshape(6, 6), oracle.stiffness(P.pagano(), 0.6),
                               atol=1e-14)


def test_bracket_parameters_known_values():
    """test_voigt_free.cpp:77-88."""
    out = (ctypes.c_double * 9)()
    assert lf.library().lf_bracket_parameters(ctypes.byref(abi.Orthotropic(*P.pagano())), out) == 0
    b = np.array(out)
    np.testing.assert_allclose(b[0], 0.07114093959731704, rtol=1e-11)
    np.testing.assert_allclose(b[1], 0.5, rtol=1e-12)
    np.testing.assert_allclose(b[2:], [24.767785234899335, -0.4, -0.3, 0, 0.2644295302013404,
                                       0.2, -0.2], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(b, SUMMARY["known_answers"]["bracket_pagano"], rtol=1e-12, atol=1e-13)


def test_angle_decomposition_matches_reference():
    out = (ctypes.c_double * 180)()
    assert lf.library().lf_angle_decomposition(ctypes.byref(abi.Orthotropic(*P.pagano())), out) == 0
    np.testing.assert_allclose(np.array(out).reshape(5, 6, 6),
                               SUMMARY["known_answers"]["angle_decomposition_pagano"], atol=1e-11)


def test_layup_dedup():
    """test_materials.cpp:170-224: cross-ply -> 2 configs, quad-ply -> 4."""
    lib = lf.library()
    for prob, want in ((P.baseline_config("C2"), 2), (P.baseline_config("C3"), 4),
                       (P.baseline_config("C4"), 3), (P.baseline_config("C5"), 4)):
        c = prob.to_c()
        n = ctypes.c_int32()
        ids = (ctypes.c_int32 * prob.n_layers)()
        assert lib.lf_layup_configs(ctypes.byref(c), ctypes.byref(n), ids, None) == 0
        assert n.value == want
        # first-appearance order
        seen = []
        for l in range(prob.n_layers):
            if prob.layers[l] not in seen:
                seen.append(prob.layers[l])
            assert ids[l] == seen.index(prob.layers[l])


def test_baseline_sizes_match_survey():
    """SURVEY.md Appendix A.1."""
    want = {"C1": (2700, 574992), "C2": (114444, 31226256), "C3": (1737243, 964255833),
            "C4": (6615180, 1924851600), "C5": (29317275, 16887368025)}
    for name, (dim, nnz) in want.items():
        prob = P.baseline_config(name)
        assert lf.pattern_size(prob) == (dim, nnz)
        assert P.sizes(prob)["nnz"] == nnz


def test_pattern_size_matches_oracle_counts(oracle):
    for prob in (P.baseline_config("C1"), P.cube_problem(3, 2, 1, [0.0, 0.5]),
                 P.baseline_config("C1").replace(active_layers=[0, 3])):
        for b in ("fast", "standard"):
            rp, _, _ = oracle.assemble(prob, b)
            assert lf.pattern_size(prob, b) == (prob.dim, int(rp[-1]))


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_slab_bounds_tile_rows_and_balance(parts):
    prob = P.baseline_config("C5")
    dim, nnz = lf.pattern_size(prob)
    prev_t, prev_r, prev_z = 0, 0, 0
    sizes = []
    for k in range(parts):
        b = lf.slab_bounds(prob, parts, k)
        assert b["t_begin"] == prev_t and b["row_begin"] == prev_r and b["nnz_begin"] == prev_z
        prev_t, prev_r, prev_z = b["t_end"], b["row_end"], b["nnz_end"]
        sizes.append(b["nnz_end"] - b["nnz_begin"])
    assert (prev_t, prev_r, prev_z) == (prob.n_t, dim, nnz)
    assert max(sizes) / (nnz / parts) < 1.05


def test_error_mapping():
    bad_knots = P.baseline_config("C1").replace(knots_u=np.array([0.0, 0.5, 1.0, 1.0, 1.0, 1.0]))
    with pytest.raises(lf.LamfastError) as e:
        lf.pattern_size(bad_knots)
    assert e.value.kind == "invalid_argument"
    bad_ifc = P.baseline_config("C1").replace(interfaces=np.array([0.0, 0.5, 0.4, 0.9, 1.0]))
    with pytest.raises(lf.LamfastError) as e:
        lf.pattern_size(bad_ifc)
    assert e.value.kind == "invalid_argument"
    bad_mat = P.baseline_config("C1").replace(layers=[(P.orthotropic(-1, 1, 1, 1, 1, 1, 0, 0, 0), 0.0)] * 4)
    with pytest.raises(lf.LamfastError) as e:
        lf.pattern_size(bad_mat)
    assert e.value.kind == "invalid_argument"
    with pytest.raises(lf.LamfastError) as e:
        lf.pattern_size(P.cube_problem(1, 1, 1, [0.0]).replace(direction=(1.0, 0.0, 0.0)))
    assert e.value.kind == "domain_error"
    with pytest.raises(lf.LamfastError) as e:
        lf.pattern_size(P.baseline_config("C1").replace(knots_u=P.uniform_knots(7, 2), degree_u=7))
    assert e.value.kind == "unsupported"


def test_mt19937_matches_std():
    """std::mt19937 default seed 5489: the 10000th output is 4123659995 (C++11 standard)."""
    rng = P.MT19937(5489)
    out = [rng() for _ in range(10000)]
    assert out[0] == 3499211612
    assert out[-1] == 4123659995


def test_baseline_layups():
    c4 = P.baseline_config("C4")
    assert c4.distinct_configs() == 3 and c4.n_layers == 128
    assert c4.layers[1][0] == P.isotropic(0.5, 0.3) and c4.layers[2][1] == P.DEG90
    c5 = P.baseline_config("C5")
    assert c5.distinct_configs() == 4 and c5.n_layers == 128
    assert P.baseline_config("C2").layers[7][1] == P.DEG90 and P.baseline_config("C2").layers[8][1] == P.DEG90


def test_c0_knots_align_with_interfaces():
    kt = P.c0_knots(2, 128)
    ifc = P.equal_interfaces(128)
    interior = kt[3:-3:2]
    assert np.array_equal(interior, ifc[1:-1])  # bit-identical: no sliver cells


def test_report_format_round_trip():
    """Reference report shape (bench.cpp:245-299), extended columns appended."""
    from paper_1905_05417_b200 import report as R
    rep = R.Report([R.Record("fast", 2, 8, 4, 2, 1.5e-5, 574992, 1e-16, 256, 8, 3.8e10, 0.05),
                    R.Record("standard", 2, 8, 4, 2, 1e-3, 574992, None, 6912, 8, 5.7e8, 0.0007)],
                   ["C9 backend=fast: boom"], 1)
    csv = R.emit_csv(rep)
    lines = csv.strip().splitlines()
    assert lines[0] == "backend,p,elements,m,m_bar,time_s,nnz,rel_diff,qpoints,elements_y,nnz_per_s,hbm_frac"
    assert lines[2].split(",")[7] == ""  # empty rel_diff cell when unavailable
    back = R.parse_json(R.emit_json(rep))
    assert back == rep


@pytest.mark.parametrize("name,parts", [("C5", 8), ("C5", 3), ("C4", 8), ("C2", 7)])
def test_function_slab_bounds_balance_and_oracle_offsets(oracle, name, parts):
    """lf_slab_bounds_functions (host only): the parts tile [0, n_t n_s),
    their nnz are balanced to within one function's row block (C5 x 8: the
    thickness-function cuts of round 1 had max/mean 1.069), and every cut's
    global offset equals the oracle's row offset of that function."""
    import paper_1905_05417_b200 as lf
    prob = P.baseline_config(name)
    terms = oracle.fast_terms(prob, want_values=False)
    prev, nnz = 0, []
    for part in range(parts):
        b = lf.slab_bounds_functions(prob, parts, part)
        assert b["f_begin"] == prev and b["f_end"] >= b["f_begin"]
        assert b["row_begin"] == 3 * b["f_begin"] and b["row_end"] == 3 * b["f_end"]
        assert b["nnz_begin"] == terms.function_offset(b["f_begin"])
        assert b["nnz_end"] == terms.function_offset(b["f_end"])
        nnz.append(b["nnz_end"] - b["nnz_begin"])
        prev = b["f_end"]
    assert prev == prob.n_s * prob.n_t
    assert sum(nnz) == P.sizes(prob)["nnz"]
    # within one function's row block (3 rows of at most 3 (2p+1)^2 L_t entries)
    assert max(nnz) - sum(nnz) / parts <= 9 * 49 * 5
    if name == "C5":
        assert max(nnz) / (sum(nnz) / parts) <= 1.000001
    terms.close()


@pytest.mark.parametrize("case", ["C1", "C2", "mixed", "masked-standard", "range"])
def test_host_pattern_columns_match_oracle(oracle, case):
    """lf_pattern_columns (host-written closed-form columns, what one-shot
    calls into host arrays use instead of copying the device pattern) equals
    the oracle's CSR columns, bit for bit."""
    backend, f0, f1 = "fast", 0, -1
    if case in ("C1", "C2"):
        prob = P.baseline_config(case)
    elif case == "mixed":
        prob = P.LaminateProblem(
            degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3), knots_v=P.uniform_knots(3, 2),
            knots_t=P.c0_knots(2, 3), interfaces=P.equal_interfaces(3),
            layers=[(P.baseline_orthotropic(), 0.0), (P.isotropic(0.5, 0.3), 0.0), (P.baseline_orthotropic(), 0.6)])
    elif case == "masked-standard":
        prob, backend = P.baseline_config("C1").replace(active_layers=[0, 3]), "standard"
    else:
        prob = P.baseline_config("C2")
        f0, f1 = prob.n_s + 5, 4 * prob.n_s - 7
    rp, cols, _ = oracle.assemble(prob, backend)
    got = lf.pattern_columns(prob, f0, f1, backend)
    if f1 < 0:
        want = cols
    else:
        want = cols[rp[3 * f0]:rp[3 * f1]]
    assert got.dtype == np.int32 and np.array_equal(got, want)


def _active_terms_per_row(prob, n_terms_of_layer):
    """Terms under each thickness function: the layers of the cells (knot span
    x ply) inside the function's support (fast.cpp:241-258)."""
    kt = np.asarray(prob.knots_t, dtype=float)
    p = prob.degree_t
    itf = np.asarray(prob.interfaces, dtype=float)
    n_t = len(kt) - p - 1
    rows = [set() for _ in range(n_t)]
    spans = [j for j in range(p, len(kt) - p - 1) if kt[j + 1] > kt[j]]
    for j in spans:
        for l in range(len(itf) - 1):
            lo, hi = max(kt[j], itf[l]), min(kt[j + 1], itf[l + 1])
            if hi - lo > 1e-14:
                for i in range(j - p, j + 1):
                    rows[i].add(n_terms_of_layer[l])
    return rows


@pytest.mark.parametrize("case", ["C2", "16 angles C0", "6 angles C1", "8 angles C2 cubic"])
def test_slot_schedule_of_the_combine(case):
    """lf_operator_terms' slot schedule (host logic of k_combine_slots): every
    term under a thickness function holds exactly one slot in that row, no
    other term is scheduled, and a term keeps its slot over consecutive rows
    (one refill per ply with one C0 element per ply)."""
    ortho = P.baseline_orthotropic()
    if case == "C2":
        prob, want_slots = P.baseline_config("C2"), 2
    elif case == "16 angles C0":
        prob, want_slots = P.plate(2, 3, 3, [(ortho, -1.5 + 0.2 * k) for k in range(16)]), 2
    elif case == "6 angles C1":
        prob = P.plate(2, 3, 3, [(ortho, -1.2 + 0.5 * (k % 6)) for k in range(9)], thickness_knots=P.uniform_knots(2, 9))
        want_slots = 3
    else:
        prob = P.plate(2, 3, 3, [(ortho, 0.25 * k) for k in range(8)], thickness_degree=3,
                       thickness_knots=P.uniform_knots(3, 8))
        want_slots = None
    tables, sched = lf.operator_terms(prob)
    seen = []  # configurations in first-appearance order (materials.cpp:203-224), as distinct_configs counts
    term_of_layer = []
    for layer in prob.layers:
        if layer not in seen:
            seen.append(layer)
        term_of_layer.append(seen.index(layer))
    assert tables.shape == (prob.distinct_configs(), 81)
    if want_slots is None:
        assert sched is None
        return
    assert sched.shape == (prob.n_t, want_slots)
    want = _active_terms_per_row(prob, term_of_layer)
    refills = 0
    held = [-1] * want_slots
    for i in range(prob.n_t):
        got = [t for t in sched[i] if t >= 0]
        assert sorted(got) == sorted(want[i]), (i, got, want[i])
        for k, t in enumerate(sched[i]):
            if t >= 0 and held[k] != t:
                held[k] = int(t)
                refills += 1
    if case == "16 angles C0":
        assert refills == len(prob.layers)  # one per ply


def test_decompose_angles_terms_fold_per_configuration_on_affine_maps():
    """setup.cpp: with a constant frame the five basis tables per material are
    summed per ply configuration, table(config) = sum_k w_k(angle) basis_k,
    which equals the directly rotated configuration's table to rounding; a
    non-affine map keeps five terms per material (fast.cpp:285-336)."""
    base = P.baseline_config("C2")
    prob = base.replace(layers=[(P.isotropic(0.5, 0.3), 0.0) if k % 3 == 1 else l for k, l in enumerate(base.layers)])
    direct, _ = lf.operator_terms(prob)
    folded, sched = lf.operator_terms(prob.replace(decompose_angles=True))
    assert direct.shape == folded.shape == (3, 81) and sched is not None
    assert np.abs(folded - direct).max() <= 1e-13 * np.abs(direct).max()
    lx, ly = prob.geometry[0], prob.geometry[1]
    skew = prob.replace(geometry_kind=1, geometry=(0, 0, 0, lx, 0.05 * ly, 0.0, -0.05 * lx, ly, 0.0,
                                                   1.02 * lx, 1.03 * ly, 0.01), decompose_angles=True)
    unfolded, _ = lf.operator_terms(skew)
    assert unfolded.shape == (10, 81)

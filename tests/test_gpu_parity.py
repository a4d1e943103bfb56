"""GPU parity: the CUDA path through the C ABI against the CPU oracle.

Gate (BASELINE.json north star): CSR pattern bit-exact; values within
1e-12 * max|K_oracle|; frobeniusRelDiff <= 1e-12 (acceptance.cpp:113).
"""
import numpy as np
import pytest

from conftest import assert_csr_match
from oracle.checkers import csr_rel_diff
from paper_1905_05417_b200 import problem as P

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def test_c1_fast_matches_oracle(gpu, oracle):
    prob = P.baseline_config("C1")
    got = gpu.assemble_fast(prob)
    want = oracle.assemble(prob, "fast")
    assert_csr_match(got.astuple(), want, RTOL)
    assert csr_rel_diff(got.astuple(), want) <= RTOL


def test_c2_fast_matches_oracle(gpu, oracle):
    prob = P.baseline_config("C2")
    got = gpu.assemble_fast(prob)
    want = oracle.assemble(prob, "fast")
    assert_csr_match(got.astuple(), want, RTOL)


def test_c1_standard_matches_oracle_and_fast(gpu, oracle):
    prob = P.baseline_config("C1")
    std = gpu.assemble_standard(prob)
    assert_csr_match(std.astuple(), oracle.assemble(prob, "standard"), RTOL)
    fast = gpu.assemble_fast(prob)
    assert np.array_equal(std.cols, fast.cols)
    assert csr_rel_diff(std.astuple(), fast.astuple()) <= RTOL


def test_c1_voigt_free_matches_fast(gpu, oracle):
    prob = P.baseline_config("C1")
    vf = gpu.assemble_voigt_free(prob)
    assert_csr_match(vf.astuple(), oracle.assemble(prob, "fast"), 1e-12)


@pytest.mark.parametrize("degree,elems,angles,geom", [
    (1, 1, [0.0], "flat"),
    (2, 2, [0.0, 1.5707963267948966, 0.0], "skewed"),
    (3, 2, [0.0, 0.7853981633974483, -0.7853981633974483, 1.5707963267948966], "flat"),
])
def test_reference_fast_equals_standard_cases(gpu, oracle, degree, elems, angles, geom):
    """test_fast.cpp:310-333 on the GPU, each backend against the oracle."""
    prob = P.cube_problem(degree, elems, 1, angles, geometry=geom)
    fast = gpu.assemble_fast(prob)
    std = gpu.assemble_standard(prob)
    vf = gpu.assemble_voigt_free(prob)
    assert_csr_match(fast.astuple(), oracle.assemble(prob, "fast"), RTOL)
    assert_csr_match(std.astuple(), oracle.assemble(prob, "standard"), RTOL)
    assert fast.nnz == std.nnz
    assert csr_rel_diff(fast.astuple(), std.astuple()) <= RTOL
    assert csr_rel_diff(vf.astuple(), std.astuple()) <= RTOL


def test_mixed_degrees_and_c0_thickness(gpu, oracle):
    """Shapes no reference test covers (SURVEY.md §4 gaps): p_u != p_v != p_t,
    C0 thickness knots, non-square plate, skewed geometry."""
    prob = P.LaminateProblem(
        degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3),
        knots_v=P.uniform_knots(3, 2), knots_t=P.c0_knots(2, 3),
        interfaces=P.equal_interfaces(3),
        layers=[(P.baseline_orthotropic(), 0.0), (P.isotropic(0.5, 0.3), 0.0),
                (P.baseline_orthotropic(), 0.6)])
    for geom in ("flat", "skewed"):
        if geom == "skewed":
            prob = prob.replace(geometry_kind=1,
                                geometry=(0, 0, 0, 1.2, 0.1, 0.05, -0.1, 0.9, -0.02, 1.0, 1.1, 0.08),
                                direction=(0.03, -0.02, 0.2))
        for backend in ("fast", "standard"):
            got = gpu.assemble_with(backend, prob)
            assert_csr_match(got.astuple(), oracle.assemble(prob, backend), RTOL)


def test_active_layers_patterns(gpu, oracle):
    """Standard drops thickness spans whose cells are all masked; fast keeps
    the full pattern (assembly.cpp:82-84 vs fast.cpp:203)."""
    prob = P.baseline_config("C1").replace(active_layers=[1])
    for backend in ("fast", "standard"):
        got = gpu.assemble_with(backend, prob)
        assert_csr_match(got.astuple(), oracle.assemble(prob, backend), RTOL)
    assert gpu.pattern_size(prob, "standard")[1] < gpu.pattern_size(prob, "fast")[1]


def test_layer_restriction_is_additive(gpu):
    """test_fast.cpp:377-388: sum over single-layer assemblies equals the whole."""
    prob = P.cube_problem(2, 2, 1, [0.0, 0.9, 0.3], geometry="skewed")
    whole = gpu.assemble_fast(prob)
    x = np.random.default_rng(31).uniform(-1, 1, whole.dim)
    import scipy.sparse as sp
    K = sp.csr_matrix((whole.values, whole.cols, whole.row_ptr), shape=(whole.dim,) * 2)
    acc = np.zeros(whole.dim)
    for l in range(3):
        part = gpu.assemble_fast(prob.replace(active_layers=[l]))
        acc += sp.csr_matrix((part.values, part.cols, part.row_ptr), shape=(whole.dim,) * 2) @ x
    y = K @ x
    assert np.linalg.norm(y - acc) <= 1e-13 * np.linalg.norm(y)


def test_decompose_angles(gpu, oracle):
    """test_fast.cpp:390-408: five builds per material; equals direct."""
    rng = P.MT19937(99)
    angles = [-1.6 + 3.2 * (rng() / 2**32) for _ in range(9)]
    prob = P.cube_problem(2, 2, 1, angles, geometry="skewed")
    direct = gpu.assemble_fast(prob)
    assert direct.stats.operator_builds == 9
    dec = gpu.assemble_fast(prob.replace(decompose_angles=True))
    assert dec.stats.operator_builds == 5
    assert csr_rel_diff(dec.astuple(), direct.astuple()) <= 1e-12
    assert_csr_match(dec.astuple(), oracle.assemble(prob.replace(decompose_angles=True), "fast"), 1e-12)


def test_many_terms_multi_pass(gpu, oracle):
    """More than 8 operator terms: the coefficient form of K4 on affine maps,
    the accumulate passes on general (skewed) ones."""
    angles = [0.1 * k for k in range(11)]
    for geom in ("flat", "skewed"):
        prob = P.cube_problem(2, 2, 2, angles, geometry=geom)
        got = gpu.assemble_fast(prob)
        assert got.stats.operator_builds == 11
        assert_csr_match(got.astuple(), oracle.assemble(prob, "fast"), RTOL)


@pytest.mark.parametrize("min_terms", ["9", "1"])
@pytest.mark.parametrize("case", ["16 angles", "decompose C2", "mixed C0", "slab"])
def test_coefficient_form_matches_oracle(gpu, oracle, monkeypatch, min_terms, case):
    """The coefficient form of the combine (one pass, 9 FMA per value for any
    term count; default from 9 terms, forced for every term count with
    LAMFAST_EFORM_MIN_TERMS=1) against the oracle: a 16-distinct-angle
    laminate, decompose_angles with two materials (10 terms), mixed degrees
    with C0 thickness knots, and a row slab cut inside a thickness row."""
    import torch
    monkeypatch.setenv("LAMFAST_EFORM_MIN_TERMS", min_terms)
    monkeypatch.setenv("LAMFAST_SLOTS_MIN_TERMS", "1000")  # not the slot form (test_slot_form_matches_oracle)
    monkeypatch.setenv("LAMFAST_FOLD_DECOMPOSE", "0")  # keep the five terms per material (test_decompose_angles_folded)
    if case == "16 angles":
        prob = P.plate(2, 6, 5, [(P.baseline_orthotropic(), -1.5 + 0.2 * k) for k in range(16)], thickness=0.2)
    elif case == "decompose C2":
        base = P.baseline_config("C2")
        layers = [(P.isotropic(0.5, 0.3), 0.0) if k % 3 == 1 else l for k, l in enumerate(base.layers)]
        prob = base.replace(layers=layers, decompose_angles=True)
    elif case == "mixed C0":
        prob = P.LaminateProblem(
            degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3),
            knots_v=P.uniform_knots(3, 2), knots_t=P.c0_knots(2, 3), interfaces=P.equal_interfaces(3),
            layers=[(P.baseline_orthotropic(), 0.0), (P.isotropic(0.5, 0.3), 0.0),
                    (P.baseline_orthotropic(), 0.6)])
    else:
        prob = P.plate(2, 6, 5, [(P.baseline_orthotropic(), -1.5 + 0.2 * k) for k in range(12)], thickness=0.2)
        ns = prob.n_s
        f0, f1 = ns + 5, 4 * ns - 7
        plan = gpu.Plan(prob, "fast", 0, f_begin=f0, f_end=f1)
        rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
        cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
        vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
        plan.build_pattern(rp.data_ptr(), cols.data_ptr())
        plan.assemble(vals.data_ptr())
        plan.synchronize()
        trp, tc, tv = oracle.assemble(prob, "fast", 1, 4)
        a, e = 3 * (f0 - ns), 3 * (f1 - ns)
        want = (trp[a:e + 1] - trp[a], tc[trp[a]:trp[e]], tv[trp[a]:trp[e]])
        assert_csr_match((rp.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy()), want, RTOL)
        plan.close()
        return
    got = gpu.assemble_fast(prob)
    assert_csr_match(got.astuple(), oracle.assemble(prob, "fast"), RTOL)


@pytest.mark.parametrize("min_terms", ["5", "1"])
@pytest.mark.parametrize("case", ["16 angles", "6 angles C1", "mixed C0", "C2", "thick p3", "slab", "too many"])
def test_slot_form_matches_oracle(gpu, oracle, monkeypatch, capfd, min_terms, case):
    """The slot form of the per-term combine (k_combine_slots: the entry's nine
    2D integrals and 2-3 register slots of P, refilled when a row brings a new
    term; default from 5 terms where every thickness row sees <= 3, forced for
    every term count with LAMFAST_SLOTS_MIN_TERMS=1) against the oracle:
    16 distinct angles with one C0 element per ply (2 slots), 6 angles on C1
    thickness splines (three plies under a function, 3 slots), mixed degrees
    and materials, BASELINE C2, cubic thickness, a row slab cut inside
    thickness rows, and a laminate whose rows see more than 3 terms (the plan
    must fall back to another form)."""
    import torch
    monkeypatch.setenv("LAMFAST_SLOTS_MIN_TERMS", min_terms)
    monkeypatch.setenv("LAMFAST_DEBUG_FORM", "1")
    ortho = P.baseline_orthotropic()
    expect = "slots"
    if case == "16 angles":
        prob = P.plate(2, 6, 5, [(ortho, -1.5 + 0.2 * k) for k in range(16)], thickness=0.2)
    elif case == "6 angles C1":
        prob = P.plate(2, 5, 4, [(ortho, -1.2 + 0.5 * (k % 6)) for k in range(9)], thickness=0.2,
                       thickness_knots=P.uniform_knots(2, 9))
    elif case == "mixed C0":
        prob = P.LaminateProblem(
            degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3),
            knots_v=P.uniform_knots(3, 2), knots_t=P.c0_knots(2, 3), interfaces=P.equal_interfaces(3),
            layers=[(ortho, 0.0), (P.isotropic(0.5, 0.3), 0.0), (ortho, 0.6)])
        if min_terms == "5":
            expect = "per-term"  # 3 terms: below the default threshold
    elif case == "C2":
        prob = P.baseline_config("C2")
        if min_terms == "5":
            expect = "per-term"
    elif case == "thick p3":
        prob = P.plate(2, 4, 4, [(ortho, 0.3 * k) for k in range(7)], thickness=0.3, thickness_degree=3,
                       thickness_knots=P.c0_knots(3, 7))
    elif case == "too many":
        # cubic C2 thickness splines: four plies under a function, each at its own angle
        prob = P.plate(2, 4, 4, [(ortho, 0.25 * k) for k in range(8)], thickness=0.2, thickness_degree=3,
                       thickness_knots=P.uniform_knots(3, 8))
        expect = "coefficient" if min_terms == "5" else None  # 8 terms: coefficient form by default
    else:
        prob = P.plate(2, 6, 5, [(ortho, -1.5 + 0.2 * k) for k in range(12)], thickness=0.2)
        ns = prob.n_s
        f0, f1 = ns + 5, 4 * ns - 7
        plan = gpu.Plan(prob, "fast", 0, f_begin=f0, f_end=f1)
        assert "combine form slots" in capfd.readouterr().err
        rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
        cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
        vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
        plan.build_pattern(rp.data_ptr(), cols.data_ptr())
        plan.assemble(vals.data_ptr())
        plan.synchronize()
        trp, tc, tv = oracle.assemble(prob, "fast", 1, 4)
        a, e = 3 * (f0 - ns), 3 * (f1 - ns)
        want = (trp[a:e + 1] - trp[a], tc[trp[a]:trp[e]], tv[trp[a]:trp[e]])
        assert_csr_match((rp.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy()), want, RTOL)
        plan.close()
        return
    capfd.readouterr()
    got = gpu.assemble_fast(prob)
    err = capfd.readouterr().err
    if expect == "slots":
        assert "combine form slots" in err, err
    elif expect is not None:
        assert f"combine form {expect}" in err and "combine form slots" not in err, err
    else:
        assert "combine form slots" not in err, err
    assert_csr_match(got.astuple(), oracle.assemble(prob, "fast"), RTOL)


@pytest.mark.parametrize("case", ["C2 with interlayers", "16 angles", "one ply active"])
def test_decompose_angles_folded_on_affine_maps(gpu, oracle, case):
    """decompose_angles on a constant frame: the five basis tables of a
    material are summed per distinct ply configuration before the combine
    (setup.cpp), so the combine runs with the direct form's terms (per-term
    kernel for <= 4 configurations, slot form above) while the work counters
    still report five builds per material (fast.cpp:285-336).  Values against
    the oracle's decomposed assembly and against the direct assembly."""
    ortho = P.baseline_orthotropic()
    if case == "C2 with interlayers":
        base = P.baseline_config("C2")
        prob = base.replace(layers=[(P.isotropic(0.5, 0.3), 0.0) if k % 3 == 1 else l
                                    for k, l in enumerate(base.layers)])
        form, builds = "per-term", 10
    elif case == "16 angles":
        prob = P.plate(2, 6, 5, [(ortho, -1.5 + 0.2 * k) for k in range(16)], thickness=0.2)
        form, builds = "slots", 5
    else:
        prob = P.plate(2, 5, 5, [(ortho, 0.4 * k) for k in range(6)], thickness=0.2).replace(active_layers=[2])
        form, builds = "slots", 5
    dec_prob = prob.replace(decompose_angles=True)
    plan = gpu.Plan(dec_prob, "fast", 0)
    assert plan.combine_form == form
    assert plan.stats().operator_builds == builds
    plan.close()
    dec = gpu.assemble_fast(dec_prob)
    assert dec.stats.operator_builds == builds
    assert_csr_match(dec.astuple(), oracle.assemble(dec_prob, "fast"), RTOL)
    assert csr_rel_diff(dec.astuple(), gpu.assemble_fast(prob).astuple()) <= 1e-12


def test_slot_form_voigt_free_backend(gpu, oracle):
    """The Voigt-free backend (contraction tables from the bracket fit,
    voigt_free.cpp:142-298) runs the same combine kernels: 16 distinct angles
    take the slot form there too."""
    prob = P.plate(2, 5, 4, [(P.baseline_orthotropic(), -1.5 + 0.2 * k) for k in range(16)], thickness=0.2)
    plan = gpu.Plan(prob, "voigt_free", 0)
    assert plan.combine_form == "slots"
    plan.close()
    got = gpu.assemble_with("voigt_free", prob)
    assert_csr_match(got.astuple(), oracle.assemble(prob, "voigt_free"), RTOL)
    assert csr_rel_diff(got.astuple(), gpu.assemble_fast(prob).astuple()) <= 1e-12


def test_stats_counters(gpu):
    """test_fast.cpp:335-352 work accounting."""
    angles = [0.0 if l % 2 == 0 else 1.5707963267948966 for l in range(32)]
    prob = P.cube_problem(3, 2, 1, angles)
    fast = gpu.assemble_fast(prob)
    assert fast.stats.operator_builds == 2
    assert fast.stats.qpoint_visits == 2 * 4 * 16
    std = gpu.assemble_standard(prob)
    assert std.stats.qpoint_visits == 32 * 4 * 16 * 4


def test_inplane_operators_match_reference(gpu, reference):
    """test_fast.cpp:278-289: P against the reference on skewed geometry,
    4 in-plane points, p_u=2, p_v=3, theta=0.6."""
    prob = P.LaminateProblem(
        degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3),
        knots_v=P.uniform_knots(3, 2), knots_t=P.uniform_knots(2, 1),
        interfaces=P.equal_interfaces(1), layers=[(P.pagano(), 0.0)],
        geometry_kind=1, geometry=(0, 0, 0, 1.2, 0.1, 0.05, -0.1, 0.9, -0.02, 1.0, 1.1, 0.08),
        direction=(0.03, -0.02, 0.2), inplane_points=4)
    d = reference.stiffness(P.pagano(), 0.6)
    got, gflags, _ = gpu.compute_inplane_operators(prob, d)
    want, wflags = reference.inplane_operators(prob, d)
    assert np.array_equal(gflags, wflags)
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()


def test_inplane_operators_affine_and_corner_block(gpu):
    """test_fast.cpp:268-276: P22(0,0) = diag(1/18, 1/18, 1/9)."""
    prob = P.cube_problem(1, 1, 1, [0.0], thickness=1.0, material=P.isotropic(1.0, 0.0))
    d = np.diag([1, 1, 1, 0.5, 0.5, 0.5]).astype(float)
    blocks, flags, _ = gpu.compute_inplane_operators(prob, d)
    # slot of (0, 0): dv = 0 + p_v, du = 0 + p_u in the band
    b = blocks[3, 0, 1, 1]
    assert np.abs(b - np.diag([1 / 18, 1 / 18, 1 / 9])).max() <= 1e-15


def test_thickness_operators_closed_form(gpu):
    """test_fast.cpp:171-188."""
    q, occ = gpu.compute_thickness_operators(1, P.uniform_knots(1, 1), [0.0, 1.0], 2)
    fam = q[0]
    assert np.abs(fam[0] - [[1 / 3, 1 / 6], [1 / 6, 1 / 3]]).max() <= 1e-15
    assert np.abs(fam[1] - [[-0.5, 0.5], [-0.5, 0.5]]).max() <= 1e-15
    assert np.abs(fam[2] - [[-0.5, -0.5], [0.5, 0.5]]).max() <= 1e-15
    assert np.abs(fam[3] - [[1, -1], [-1, 1]]).max() <= 1e-15
    assert occ[0, 1] == 1


def test_thickness_operators_match_reference(gpu, reference):
    kt = P.uniform_knots(3, 2)
    ifc = [0.0, 0.2, 0.5, 0.7, 1.0]
    got, gocc = gpu.compute_thickness_operators(3, kt, ifc, 4)
    want, wocc = reference.thickness_operators(3, kt, ifc, 4)
    assert np.array_equal(gocc, wocc)
    assert np.abs(got - want).max() <= 1e-15
    assert gocc[0, 4] == 0 and gocc[1, 4] == 1


def test_combine_operators_long_form(gpu, oracle):
    """test_fast.cpp:354-375: per-layer long form == pre-reduced q~."""
    prob = P.cube_problem(2, 2, 2, [0.0, 1.5707963267948966, 1.5707963267948966, 0.0],
                          lx=1.3, ly=0.8, thickness=0.2)
    reduced = gpu.assemble_fast(prob)
    q, occ = gpu.compute_thickness_operators(2, prob.knots_t, prob.interfaces, 3)
    sets = {}
    for c, a in prob.layers:
        if a not in sets:
            d = oracle.stiffness(c, a)
            sets[a] = gpu.compute_inplane_operators(prob, d)
    blocks = np.stack([sets[a][0] for _, a in prob.layers])
    flags = sets[prob.layers[0][1]][1]
    long_form = gpu.combine_operators(prob, blocks, flags, q, occ)
    assert long_form.nnz == reduced.nnz
    assert csr_rel_diff(long_form.astuple(), reduced.astuple()) <= 1e-14


def test_degenerate_geometry_raises_domain_error(gpu):
    prob = P.cube_problem(1, 1, 1, [0.0]).replace(direction=(1.0, 0.0, 0.0))
    with pytest.raises(gpu.LamfastError) as e:
        gpu.assemble_fast(prob)
    assert e.value.kind == "domain_error"


def test_row_slabs_match_oracle_slabs(gpu, oracle):
    """Slab plans (the multi-GPU unit) against oracle slab mode."""
    import torch
    prob = P.baseline_config("C2")
    for parts in (2, 3):
        for part in range(parts):
            b = gpu.slab_bounds(prob, parts, part)
            plan = gpu.Plan(prob, "fast", 0, b["t_begin"], b["t_end"])
            rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
            cols = torch.empty(max(1, plan.nnz), dtype=torch.int32, device="cuda")
            vals = torch.empty(max(1, plan.nnz), dtype=torch.float64, device="cuda")
            plan.build_pattern(rp.data_ptr(), cols.data_ptr())
            plan.assemble(vals.data_ptr())
            plan.synchronize()
            want = oracle.assemble(prob, "fast", b["t_begin"], b["t_end"])
            assert_csr_match((rp.cpu().numpy(), cols.cpu().numpy()[:plan.nnz],
                              vals.cpu().numpy()[:plan.nnz]), want, RTOL)
            plan.close()


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_config_slab_and_properties(gpu, oracle, name):
    """BASELINE C3/C4 at full size on the device: an oracle-checked slab,
    plus size-independent properties of the whole matrix (rigid
    translations annihilated, symmetry, nnz)."""
    import torch
    prob = P.baseline_config(name)
    plan = gpu.Plan(prob, "fast", 0)
    assert plan.nnz == P.sizes(prob)["nnz"]
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    # slab check: rows of thickness functions [t, t+3) from the middle
    t = prob.n_t // 2
    want = oracle.assemble(prob, "fast", t, t + 3)
    r0 = 3 * prob.n_s * t
    r1 = 3 * prob.n_s * (t + 3)
    z0, z1 = int(rp[r0]), int(rp[r1])
    got = ((rp[r0:r1 + 1] - z0).cpu().numpy(), cols[z0:z1].cpu().numpy(), vals[z0:z1].cpu().numpy())
    assert_csr_match(got, want, RTOL)
    # translations: K t = 0 for rigid translations (acceptance.cpp:95-104)
    lib = gpu.library()
    st = gpu.device_csr_stats(plan.rows, rp.data_ptr(), cols.data_ptr(), vals.data_ptr())
    norm = np.sqrt(st["fro_sq"])
    assert np.sqrt(st["sym_sq"]) / norm <= 1e-13
    assert np.sqrt(plan.symmetry_sq(vals.data_ptr())) / norm <= 1e-13
    import ctypes
    for d in range(3):
        x = torch.zeros(plan.rows, dtype=torch.float64, device="cuda")
        x[d::3] = 1.0
        y = torch.empty_like(x)
        assert lib.lf_csr_spmv(plan.rows, ctypes.c_void_p(rp.data_ptr()), ctypes.c_void_p(cols.data_ptr()),
                               ctypes.c_void_p(vals.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                               ctypes.c_void_p(y.data_ptr()), None) == 0
        torch.cuda.synchronize()
        assert float(y.abs().max()) / norm <= 1e-12
    plan.close()


# ---- against the frozen outputs of the unmodified reference -------------------

import json as _json
import os as _os
import sys as _sys

_GOLD_DIR = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "golden")
_sys.path.insert(0, _GOLD_DIR)
from cases import cases as _cases  # noqa: E402


@pytest.mark.parametrize("name", list(_cases().keys()))
def test_gpu_matches_reference_fixtures(gpu, name):
    gold = np.load(_os.path.join(_GOLD_DIR, "ref_small.npz"))
    with open(_os.path.join(_GOLD_DIR, "ref_summaries.json")) as f:
        meta = _json.load(f)["small"]
    prob, backends = _cases()[name]
    for b in backends:
        key = f"{name}__{b}"
        want = (gold[key + "__row_ptr"], gold[key + "__cols"], gold[key + "__values"])
        got = gpu.assemble_with(b, prob)
        assert_csr_match(got.astuple(), want, RTOL)
        assert csr_rel_diff(got.astuple(), want) <= RTOL
        assert got.stats.qpoint_visits == meta[key]["qpoint_visits"]
        assert got.stats.frame_evaluations == meta[key]["frame_evaluations"]
        assert got.stats.operator_builds == meta[key]["operator_builds"]


def test_gpu_matches_reference_c1_c2_summaries(gpu):
    import hashlib
    with open(_os.path.join(_GOLD_DIR, "ref_summaries.json")) as f:
        summ = _json.load(f)["baseline"]
    for key, s in summ.items():
        name, b = key.split("__")
        got = gpu.assemble_with(b, P.baseline_config(name))
        assert hashlib.sha256(got.row_ptr.tobytes()).hexdigest() == s["row_ptr_sha256"]
        assert hashlib.sha256(got.cols.tobytes()).hexdigest() == s["cols_sha256"]
        assert np.sqrt(got.values @ got.values) == pytest.approx(s["fro"], rel=1e-13)
        idx = np.asarray(s["sample_idx"])
        assert np.abs(got.values[idx] - s["sample_values"]).max() <= RTOL * s["max_abs"]


def _device_csr(gpu, prob, backend, t0=0, t1=-1):
    import torch
    plan = gpu.Plan(prob, backend, 0, t0, t1)
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(max(1, plan.nnz), dtype=torch.int32, device="cuda")
    vals = torch.empty(max(1, plan.nnz), dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    rows = plan.rows
    plan.close()
    return rows, rp, cols, vals


def _device_rel_diff(gpu, a, b):
    import ctypes
    lib = gpu.library()
    d2, fa, fb = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())
    assert lib.lf_csr_diff_sq(a[0], ptr(a[1]), ptr(a[2]), ptr(a[3]), ptr(b[1]), ptr(b[2]), ptr(b[3]),
                              None, ctypes.byref(d2)) == 0
    assert lib.lf_csr_frobenius_sq(a[0], ptr(a[1]), ptr(a[3]), None, ctypes.byref(fa)) == 0
    assert lib.lf_csr_frobenius_sq(b[0], ptr(b[1]), ptr(b[3]), None, ctypes.byref(fb)) == 0
    return (d2.value / max(fa.value, fb.value)) ** 0.5


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_fast_equals_standard_on_device(gpu, name):
    """The paper's equivalence at BASELINE size: fast (sum-factorised P,
    Kronecker combination) vs standard (full 3D quadrature, coloured
    scatter) -- two independent device paths -- frobeniusRelDiff <= 1e-12 and
    identical patterns."""
    import torch
    prob = P.baseline_config(name)
    fast = _device_csr(gpu, prob, "fast")
    std = _device_csr(gpu, prob, "standard")
    assert torch.equal(fast[1], std[1]) and torch.equal(fast[2], std[2])
    assert _device_rel_diff(gpu, fast, std) <= RTOL
    del std
    torch.cuda.empty_cache()
    # the Voigt-free formulation (contraction tables from the bracket fit) too
    vf = _device_csr(gpu, prob, "voigt_free")
    assert torch.equal(fast[1], vf[1]) and torch.equal(fast[2], vf[2])
    assert _device_rel_diff(gpu, fast, vf) <= RTOL
    del fast, vf
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_c5_slab_fast_equals_standard_on_device(gpu):
    """C5 (203 GB CSR) cannot be resident at once: all of it, in 8 row slabs,
    fast against standard on the device -- identical patterns and
    frobeniusRelDiff <= 1e-12 over the whole matrix (slab sums)."""
    import ctypes
    import torch
    prob = P.baseline_config("C5")
    lib = gpu.library()
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())
    d2 = fa = fb = 0.0
    for part in range(8):
        b = gpu.slab_bounds(prob, 8, part)
        fast = _device_csr(gpu, prob, "fast", b["t_begin"], b["t_end"])
        std = _device_csr(gpu, prob, "standard", b["t_begin"], b["t_end"])
        assert torch.equal(fast[1], std[1]) and torch.equal(fast[2], std[2])
        x, y, z = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        assert lib.lf_csr_diff_sq(fast[0], ptr(fast[1]), ptr(fast[2]), ptr(fast[3]), ptr(std[1]), ptr(std[2]),
                                  ptr(std[3]), None, ctypes.byref(x)) == 0
        assert lib.lf_csr_frobenius_sq(fast[0], ptr(fast[1]), ptr(fast[3]), None, ctypes.byref(y)) == 0
        assert lib.lf_csr_frobenius_sq(std[0], ptr(std[1]), ptr(std[3]), None, ctypes.byref(z)) == 0
        d2, fa, fb = d2 + x.value, fa + y.value, fb + z.value
        del fast, std
        torch.cuda.empty_cache()
    assert (d2 / max(fa, fb)) ** 0.5 <= RTOL


@pytest.mark.parametrize("env", [{}, {"LAMFAST_TCHUNK": "7"}])
def test_combine_chunking_and_odd_phases_match_oracle(gpu, oracle, monkeypatch, env):
    """The combine with its default and an odd thickness chunk (7 rows) gives
    the oracle's CSR: boundary groups, mixed degrees / C0 thickness, skewed
    geometry (general P), and slab plans whose output ranges start at odd
    8-byte phases."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    mixed = P.LaminateProblem(
        degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3),
        knots_v=P.uniform_knots(3, 2), knots_t=P.c0_knots(2, 3),
        interfaces=P.equal_interfaces(3),
        layers=[(P.baseline_orthotropic(), 0.0), (P.isotropic(0.5, 0.3), 0.0),
                (P.baseline_orthotropic(), 0.6)])
    skew = P.cube_problem(2, 3, 2, [0.0, 0.9, 0.3], geometry="skewed")
    for prob in (P.baseline_config("C1"), P.baseline_config("C2"), mixed, skew):
        got = gpu.assemble_fast(prob)
        assert_csr_match(got.astuple(), oracle.assemble(prob, "fast"), RTOL)
    prob = P.baseline_config("C2")
    for part in range(3):
        b = gpu.slab_bounds(prob, 3, part)
        plan = gpu.Plan(prob, "fast", 0, b["t_begin"], b["t_end"])
        rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
        cols = torch.empty(max(1, plan.nnz), dtype=torch.int32, device="cuda")
        # values at an 8-byte (not 16-byte) aligned base: odd bulk-copy phase
        raw = torch.empty(max(1, plan.nnz) + 1, dtype=torch.float64, device="cuda")
        plan.build_pattern(rp.data_ptr(), cols.data_ptr())
        plan.assemble(raw.data_ptr() + 8)
        plan.synchronize()
        want = oracle.assemble(prob, "fast", b["t_begin"], b["t_end"])
        assert_csr_match((rp.cpu().numpy(), cols.cpu().numpy()[:plan.nnz],
                          raw.cpu().numpy()[1:plan.nnz + 1]), want, RTOL)
        plan.close()


@pytest.mark.parametrize("sym", ["1", "0"])
def test_standard_symmetric_halving_matches_oracle(gpu, oracle, monkeypatch, sym):
    """K6 computes local pairs al <= be and mirrors them when every term table
    has major symmetry; LAMFAST_NO_SYM=1 forces all pairs.  Both match the
    oracle, including a slab plan whose cut separates mirrored rows."""
    import torch
    if sym == "0":
        monkeypatch.setenv("LAMFAST_NO_SYM", "1")
    prob = P.cube_problem(2, 2, 2, [0.0, 0.9, 0.3], geometry="skewed")
    got = gpu.assemble_standard(prob)
    assert_csr_match(got.astuple(), oracle.assemble(prob, "standard"), RTOL)
    prob = P.baseline_config("C1")
    b = gpu.slab_bounds(prob, 2, 1)
    plan = gpu.Plan(prob, "standard", 0, b["t_begin"], b["t_end"])
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(max(1, plan.nnz), dtype=torch.int32, device="cuda")
    vals = torch.empty(max(1, plan.nnz), dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    want = oracle.assemble(prob, "standard", b["t_begin"], b["t_end"])
    assert_csr_match((rp.cpu().numpy(), cols.cpu().numpy()[:plan.nnz], vals.cpu().numpy()[:plan.nnz]),
                     want, RTOL)
    plan.close()


def test_concurrent_calls_are_reentrant(gpu):
    """The reference's assembly functions are pure and reentrant and may be
    called concurrently: eight host threads calling the
    C ABI at once (ctypes drops the GIL) get the bitwise results of the
    sequential calls -- every call owns its stream and device buffers."""
    import threading
    cases = [("fast", P.baseline_config("C1")), ("standard", P.baseline_config("C1")),
             ("fast", P.cube_problem(3, 2, 2, [0.0, 0.5 * P.PI, 0.25 * P.PI])),
             ("voigt_free", P.cube_problem(2, 2, 1, [0.0, 0.25 * P.PI], geometry="skewed")),
             ("fast", P.baseline_config("C2"))]
    want = [gpu.assemble_with(b, p).astuple() for b, p in cases]
    got = [None] * (2 * len(cases))
    errors = []

    def run(i):
        try:
            b, p = cases[i % len(cases)]
            got[i] = gpu.assemble_with(b, p).astuple()
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(got))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i, g in enumerate(got):
        w = want[i % len(cases)]
        for a, b in zip(g, w):
            assert np.array_equal(a, b)


def test_general_inplane_forms_match_oracle(gpu, oracle):
    """Non-affine maps take the general in-plane path (K2b, element-local P +
    gather), which matches the oracle -- degrees 1..4, mixed in-plane degrees
    (the runtime-degree gather), several terms."""
    cases = [P.cube_problem(p, 3, 1, [0.0, 0.9, 0.3, 1.2][:p + 1], geometry="skewed") for p in (1, 2, 3, 4)]
    cases.append(P.LaminateProblem(
        degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 4),
        knots_v=P.uniform_knots(3, 3), knots_t=P.c0_knots(2, 3),
        interfaces=P.equal_interfaces(3),
        layers=[(P.baseline_orthotropic(), 0.0), (P.isotropic(0.5, 0.3), 0.0),
                (P.baseline_orthotropic(), 0.6)],
        geometry_kind=1, geometry=(0, 0, 0, 1.2, 0.1, 0.05, -0.1, 0.9, -0.02, 1.0, 1.1, 0.08),
        direction=(0.03, -0.02, 0.2)))
    for prob in cases:
        got = gpu.assemble_fast(prob)
        assert_csr_match(got.astuple(), oracle.assemble(prob, "fast"), RTOL)


@pytest.mark.parametrize("p", [5, 6])
def test_maximum_supported_degrees_match_oracle(gpu, oracle, p):
    """The device tables are sized for degree <= 6 (kMaxP; degree 7 maps to
    LF_ERR_UNSUPPORTED, test_host.py): the largest degrees, in-plane and
    through the thickness, on flat and skewed maps, fast and standard."""
    for geom in ("flat", "skewed"):
        prob = P.cube_problem(p, 1, 1, [0.0, 0.7], geometry=geom)
        for backend in ("fast", "standard"):
            got = gpu.assemble_with(backend, prob)
            assert_csr_match(got.astuple(), oracle.assemble(prob, backend), RTOL)


def test_empty_and_single_row_slabs(gpu, oracle):
    """Degenerate slab plans: an empty thickness range has no rows and no
    values (row_ptr = [0]); a single thickness function's slab equals the
    oracle's rows; assembling an empty slab is a no-op."""
    import torch
    prob = P.baseline_config("C1")
    plan = gpu.Plan(prob, "fast", 0, 2, 2)
    assert plan.rows == 0 and plan.nnz == 0
    rp = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    cols = torch.empty(1, dtype=torch.int32, device="cuda")
    vals = torch.full((1,), 7.0, dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    assert int(rp[0]) == 0 and float(vals[0]) == 7.0
    plan.close()
    for t in (0, prob.n_t - 1):
        plan = gpu.Plan(prob, "fast", 0, t, t + 1)
        rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
        cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
        vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
        plan.build_pattern(rp.data_ptr(), cols.data_ptr())
        plan.assemble(vals.data_ptr())
        plan.synchronize()
        assert_csr_match((rp.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy()),
                         oracle.assemble(prob, "fast", t, t + 1), RTOL)
        plan.close()


@pytest.mark.parametrize("p", [1, 3])
def test_uniform_stretch_stores_the_axial_stiffness(gpu, p):
    """test_assembly.cpp:156-174 on the device: u(x) = x e_1 on a flat box of
    isotropic material (E = 2.3, nu = 0.28) is a uniform stretch, so
    u^T K u = (lambda + 2 mu) * volume for every backend.  p = 1 is the
    reference's unit cube (coefficients = node x-coordinates); p = 3 uses
    the Greville abscissae (linear fields are reproduced exactly) on a
    2x2-element, 3-ply box of 1.5 x 0.8 x 0.4."""
    e, nu = 2.3, 0.28
    lam = e * nu / ((1 + nu) * (1 - 2 * nu))
    mu = e / (2 * (1 + nu))
    mat = P.isotropic(e, nu)
    if p == 1:
        prob = P.cube_problem(1, 1, 1, [(mat, 0.0)], thickness=1.0)
        lx, vol = 1.0, 1.0
    else:
        lx, ly, h = 1.5, 0.8, 0.4
        prob = P.cube_problem(3, 2, 1, [(mat, 0.0), (mat, 0.7), (mat, -0.3)], lx=lx, ly=ly, thickness=h)
        vol = lx * ly * h
    ku = prob.knots_u
    greville = np.array([ku[i + 1:i + 1 + p].mean() for i in range(prob.n_u)])
    u = np.zeros(prob.dim)
    for f in range(prob.n_u * prob.n_v * prob.n_t):
        u[3 * f] = lx * greville[f % prob.n_u]
    for backend in ("fast", "standard", "voigt_free"):
        k = gpu.assemble_with(backend, prob)
        rows = np.repeat(np.arange(prob.dim), np.diff(k.row_ptr))
        ku_vec = np.bincount(rows, weights=k.values * u[k.cols], minlength=prob.dim)
        assert u @ ku_vec == pytest.approx((lam + 2 * mu) * vol, rel=1e-13)


def test_one_shot_slabs_match_oracle(gpu, oracle):
    """lf_assemble_slab (one rank's one-shot call, host buffers) returns the
    oracle's rows for every part of a 3-way split, for fast and standard;
    the parts concatenate to the whole matrix; an empty slab is row_ptr [0]."""
    import torch
    for backend in ("fast", "standard"):
        prob = P.baseline_config("C2")
        full = gpu.assemble_with(backend, prob)
        vals = []
        for part in range(3):
            b = gpu.slab_bounds(prob, 3, part, backend)
            got = gpu.assemble_slab(prob, b["t_begin"], b["t_end"], backend)
            assert_csr_match(got.astuple(), oracle.assemble(prob, backend, b["t_begin"], b["t_end"]), RTOL)
            vals.append(got.values)
        cat = np.concatenate(vals)
        if backend == "fast": # same arithmetic per value (test_slabs_are_bitwise_rows_of_the_full_matrix)
            assert np.array_equal(cat, full.values)
        else:
            assert np.abs(cat - full.values).max() <= RTOL * np.abs(full.values).max()
    pinned = (torch.empty(1, dtype=torch.int64, pin_memory=True), torch.empty(1, dtype=torch.int32, pin_memory=True),
              torch.empty(1, dtype=torch.float64, pin_memory=True))
    empty = gpu.assemble_slab(P.baseline_config("C1"), 3, 3, out=pinned)
    assert int(empty.row_ptr[0]) == 0 and empty.nnz == 0


def test_matrix_free_bilinear_matches_reference(gpu, reference):
    """lf_reference_bilinear (K8: v^T K u by full 3D quadrature, no matrix)
    equals the unmodified reference's referenceBilinear (assembly.cpp:247-318)
    and v^T K u of the device standard assembly, on flat, skewed, mixed-degree
    / C0-thickness and masked-layer problems, with random fields."""
    rng = np.random.default_rng(7)
    mixed = P.LaminateProblem(
        degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3),
        knots_v=P.uniform_knots(3, 2), knots_t=P.c0_knots(2, 3),
        interfaces=P.equal_interfaces(3),
        layers=[(P.baseline_orthotropic(), 0.0), (P.isotropic(0.5, 0.3), 0.0),
                (P.baseline_orthotropic(), 0.6)])
    cases = [P.baseline_config("C1"), P.cube_problem(2, 2, 2, [0.0, 0.9, 0.3], geometry="skewed"), mixed,
             P.cube_problem(2, 2, 1, [0.0, 0.5 * P.PI, 0.3, 1.1]).replace(active_layers=[1, 2])]
    for prob in cases:
        u = rng.standard_normal(prob.dim)
        v = rng.standard_normal(prob.dim)
        got = gpu.reference_bilinear(prob, v, u)
        want = reference.bilinear(prob, v, u)
        k = gpu.assemble_standard(prob)
        rows = np.repeat(np.arange(prob.dim), np.diff(k.row_ptr))
        vku = v @ np.bincount(rows, weights=k.values * u[k.cols], minlength=prob.dim)
        scale = np.sqrt(abs(reference.bilinear(prob, u, u) * reference.bilinear(prob, v, v)))
        assert abs(got - want) <= 1e-12 * scale
        assert abs(got - vku) <= 1e-12 * scale


@pytest.mark.slow
def test_c5_layup_reduced_inplane_matches_oracle(gpu, oracle):
    """The C5 laminate itself (128 plies, orientations from std::mt19937(20190514),
    4 distinct rotated materials, p = 3, thickness 0.25) on a 32 x 32 in-plane
    mesh, so the oracle finishes in seconds: device slab plans of three
    thickness functions at the bottom, middle and top equal the oracle's rows."""
    import torch
    c5 = P.baseline_config("C5")
    prob = P.plate(3, 32, 32, c5.layers, thickness=0.25, name="C5-32x32")
    assert prob.distinct_configs() == 4
    for t in (0, prob.n_t // 2, prob.n_t - 3):
        plan = gpu.Plan(prob, "fast", 0, t, t + 3)
        rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
        cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
        vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
        plan.build_pattern(rp.data_ptr(), cols.data_ptr())
        plan.assemble(vals.data_ptr())
        plan.synchronize()
        assert_csr_match((rp.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy()),
                         oracle.assemble(prob, "fast", t, t + 3), RTOL)
        plan.close()


@pytest.mark.slow
def test_full_size_decompose_angles_equals_direct_on_device(gpu):
    """AssemblyOptions::decompose_angles at BASELINE C3 size (4 angles of one
    material -> 5 trigonometric terms, one multi-term pass) equals the direct
    per-angle fast assembly: same pattern, frobeniusRelDiff <= 1e-12."""
    import torch
    prob = P.baseline_config("C3")
    direct = _device_csr(gpu, prob, "fast")
    dec = _device_csr(gpu, prob.replace(decompose_angles=True), "fast")
    assert torch.equal(direct[1], dec[1]) and torch.equal(direct[2], dec[2])
    assert _device_rel_diff(gpu, direct, dec) <= RTOL
    del direct, dec
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_full_size_general_geometry_fast_equals_standard_on_device(gpu):
    """C3's mesh and layup on a bilinear (non-affine) map: the general in-plane
    path (two-phase K2b, per-point frames) against the standard assembly on
    the device, at full size."""
    import torch
    prob = P.baseline_config("C3")
    prob = prob.replace(geometry_kind=1, geometry=(0, 0, 0, 1.0, 0.05, 0.0, -0.05, 1.0, 0.0, 1.02, 1.03, 0.01))
    fast = _device_csr(gpu, prob, "fast")
    std = _device_csr(gpu, prob, "standard")
    assert torch.equal(fast[1], std[1]) and torch.equal(fast[2], std[2])
    assert _device_rel_diff(gpu, fast, std) <= RTOL
    del fast, std
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_c5_full_size_rows_annihilate_translations(gpu):
    """C5 at full size (1.69e10 nnz, 203 GB as CSR -- never resident at once):
    every one of its rows, assembled slab by slab (8 row slabs, pattern and
    values each), annihilates the three rigid translations (acceptance.cpp:
    95-104) within 1e-12 of ||K||_F, the slabs' nnz add up to the closed form,
    and K is symmetric in the bilinear sense v.(K u) = u.(K v) for random u, v."""
    import ctypes
    import torch
    prob = P.baseline_config("C5")
    lib = gpu.library()
    parts, total_nnz, fro_sq, worst = 8, 0, 0.0, 0.0
    xs = []
    for d in range(3):
        x = torch.zeros(prob.dim, dtype=torch.float64, device="cuda")
        x[d::3] = 1.0
        xs.append(x)
    gen = torch.Generator(device="cuda").manual_seed(5)
    u = torch.randn(prob.dim, dtype=torch.float64, device="cuda", generator=gen)
    v = torch.randn(prob.dim, dtype=torch.float64, device="cuda", generator=gen)
    ku = torch.empty_like(u)
    kv = torch.empty_like(v)
    xs += [u, v]
    for part in range(parts):
        b = gpu.slab_bounds(prob, parts, part)
        plan = gpu.Plan(prob, "fast", 0, b["t_begin"], b["t_end"])
        rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
        cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
        vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
        plan.build_pattern(rp.data_ptr(), cols.data_ptr())
        plan.assemble(vals.data_ptr())
        plan.synchronize()
        total_nnz += plan.nnz
        f = ctypes.c_double()
        assert lib.lf_csr_frobenius_sq(plan.rows, ctypes.c_void_p(rp.data_ptr()), ctypes.c_void_p(vals.data_ptr()),
                                       None, ctypes.byref(f)) == 0
        fro_sq += f.value
        y = torch.empty(plan.rows, dtype=torch.float64, device="cuda")
        r0, r1 = b["row_begin"], b["row_end"]
        for i, x in enumerate(xs):
            assert lib.lf_csr_spmv(plan.rows, ctypes.c_void_p(rp.data_ptr()), ctypes.c_void_p(cols.data_ptr()),
                                   ctypes.c_void_p(vals.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                                   ctypes.c_void_p(y.data_ptr()), None) == 0
            torch.cuda.synchronize()
            if i < 3:
                worst = max(worst, float(y.abs().max()))
            else:
                (ku if i == 3 else kv)[r0:r1] = y
        plan.close()
        del rp, cols, vals, y
        torch.cuda.empty_cache()
    assert total_nnz == P.sizes(prob)["nnz"]
    assert worst / np.sqrt(fro_sq) <= 1e-12
    asym = abs(float(v @ ku) - float(u @ kv))
    assert asym <= 1e-12 * np.sqrt(fro_sq) * float(u.norm()) * float(v.norm())


def _host_symmetry_sq(rp, cols, vals, row_begin, dim):
    """Reference numerator (sparse.cpp:73-95) restricted to the entries of the
    slab whose mirror row lies in the slab: ||S - S^T||_F^2 of the slab's
    square in-slab block (an absent mirror contributes v^2 twice either way)."""
    import scipy.sparse as sp
    rows = len(rp) - 1
    S = sp.csr_matrix((vals, cols, rp), shape=(rows, dim))[:, row_begin:row_begin + rows].tocsr()
    D = (S - S.T).tocsr()
    return float(D.data @ D.data), int(len(vals) - S.nnz)


@pytest.mark.parametrize("parts,part", [(1, 0), (3, 0), (3, 1), (3, 2)])
def test_symmetry_sums_match_host_on_slabs(gpu, parts, part):
    """Device symmetry numerators -- the generic CSR kernel with a global row
    offset (lf_csr_symmetry_sq_slab) and the plan's closed-form kernel
    (lf_plan_symmetry_sq) -- equal the host's on a C2 row slab whose values
    carry a seeded asymmetric perturbation (a symmetric K would only compare
    roundoff); the full-matrix entry point rejects a slab."""
    import ctypes
    import torch
    prob = P.baseline_config("C2")
    lib = gpu.library()
    b = gpu.slab_bounds(prob, parts, part)
    plan = gpu.Plan(prob, "fast", 0, b["t_begin"], b["t_end"])
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    gen = torch.Generator(device="cuda").manual_seed(17 + part)
    vals += 1e-3 * vals.abs().max() * torch.rand(plan.nnz, dtype=torch.float64, device="cuda", generator=gen)
    want, skipped = _host_symmetry_sq(rp.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy(),
                                      b["row_begin"], prob.dim)
    st = gpu.device_csr_stats(plan.rows, rp.data_ptr(), cols.data_ptr(), vals.data_ptr(), row_begin=b["row_begin"])
    assert st["sym_sq"] == pytest.approx(want, rel=1e-12)
    assert st["sym_skipped"] == skipped
    assert plan.symmetry_sq(vals.data_ptr()) == pytest.approx(want, rel=1e-12)
    out = ctypes.c_double()
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())
    status = lib.lf_csr_symmetry_sq(plan.rows, ptr(rp), ptr(cols), ptr(vals), None, ctypes.byref(out))
    assert (status == 0) == (parts == 1)
    if parts == 1:
        assert out.value == pytest.approx(want, rel=1e-12)
    plan.close()


def test_symmetry_of_unperturbed_matrix_is_roundoff(gpu):
    """Both symmetry kernels on the unperturbed C2 matrix: at roundoff."""
    prob = P.baseline_config("C2")
    import torch
    plan = gpu.Plan(prob, "fast", 0)
    rows, rp, cols, vals = plan.rows, None, None, None
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    st = gpu.device_csr_stats(rows, rp.data_ptr(), cols.data_ptr(), vals.data_ptr())
    assert st["sym_sq"] ** 0.5 <= 1e-13 * st["fro_sq"] ** 0.5
    assert plan.symmetry_sq(vals.data_ptr()) ** 0.5 <= 1e-13 * st["fro_sq"] ** 0.5
    plan.close()

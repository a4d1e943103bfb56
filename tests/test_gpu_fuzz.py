"""Randomised parity: GPU (C ABI) vs the CPU oracle on random small laminates --
degrees 1..4 per direction, interior knot multiplicities up to p, non-uniform
ply interfaces (cells that cut knot spans), random materials/angles with
repeats, masked layers, decompose_angles, flat and skewed geometry."""
import numpy as np
import pytest

from conftest import assert_csr_match
from paper_1905_05417_b200 import problem as P

pytestmark = pytest.mark.gpu


def random_knots(rng, p, n_el):
    k = [0.0] * (p + 1)
    for i in range(1, n_el):
        k += [float(i) / n_el] * int(rng.integers(1, p + 1))
    return np.asarray(k + [1.0] * (p + 1))


def random_problem(seed):
    rng = np.random.default_rng(seed)
    pu, pv, pt = (int(x) for x in rng.integers(1, 5, size=3))
    m = int(rng.integers(1, 6))
    if rng.uniform() < 0.5:
        ifc = P.equal_interfaces(m)
        kt = P.c0_knots(pt, m) if rng.uniform() < 0.5 else random_knots(rng, pt, int(rng.integers(1, 4)))
    else:
        cuts = np.sort(rng.uniform(0.05, 0.95, m - 1))
        ifc = np.concatenate([[0.0], cuts, [1.0]])
        kt = random_knots(rng, pt, int(rng.integers(1, 4)))
    mats = [P.baseline_orthotropic(), P.pagano(), P.isotropic(0.5, 0.3)]
    angles = [0.0, 0.5 * P.PI, 0.25 * P.PI, float(rng.uniform(-1.5, 1.5))]
    layers = [(mats[int(rng.integers(0, 3))], angles[int(rng.integers(0, 4))]) for _ in range(m)]
    prob = P.LaminateProblem(
        degree_u=pu, degree_v=pv, degree_t=pt,
        knots_u=random_knots(rng, pu, int(rng.integers(1, 4))),
        knots_v=random_knots(rng, pv, int(rng.integers(1, 4))), knots_t=kt,
        interfaces=ifc, layers=layers, geometry=(float(rng.uniform(0.5, 2)), float(rng.uniform(0.5, 2))),
        direction=(0.0, 0.0, float(rng.uniform(0.05, 0.5))))
    if rng.uniform() < 0.4:
        prob = prob.replace(geometry_kind=1,
                            geometry=(0, 0, 0, 1.2, 0.1, 0.05, -0.1, 0.9, -0.02, 1.0, 1.1, 0.08),
                            direction=(0.03, -0.02, 0.2))
    if rng.uniform() < 0.25 and m > 1:
        prob = prob.replace(active_layers=sorted(set(int(x) for x in rng.integers(0, m, size=2))))
    if rng.uniform() < 0.2:
        prob = prob.replace(decompose_angles=True)
    if rng.uniform() < 0.2:
        prob = prob.replace(inplane_points=int(rng.integers(max(pu, pv) + 1, 7)),
                            thickness_points=int(rng.integers(pt + 1, 6)))
    return prob


@pytest.mark.parametrize("seed", range(40))
def test_random_problem_matches_oracle(gpu, oracle, seed):
    prob = random_problem(seed)
    for backend in ("fast", "standard"):
        got = gpu.assemble_with(backend, prob)
        want = oracle.assemble(prob, backend, want_stats=True)
        assert_csr_match(got.astuple(), want[:3], 1e-12)
        assert got.stats.qpoint_visits == want[3].qpoint_visits
        assert got.stats.operator_builds == want[3].operator_builds


def random_many_angle_problem(seed):
    """Flat laminates with 5..12 plies at (mostly) distinct angles over random
    thickness spaces: the slot form of the combine where every thickness row
    sees <= 3 configurations, the coefficient / per-term forms otherwise."""
    rng = np.random.default_rng(1000 + seed)
    pu, pv = (int(x) for x in rng.integers(1, 4, size=2))
    pt = int(rng.integers(1, 4))
    m = int(rng.integers(5, 13))
    r = rng.uniform()
    if r < 0.4:  # one C0 element per ply
        ifc, kt = P.equal_interfaces(m), P.c0_knots(pt, m)
    elif r < 0.7:  # one element per ply, random continuity
        ifc, kt = P.equal_interfaces(m), random_knots(rng, pt, m)
    else:  # plies that cut the knot spans
        cuts = np.sort(rng.uniform(0.05, 0.95, m - 1))
        ifc = np.concatenate([[0.0], cuts, [1.0]])
        kt = random_knots(rng, pt, int(rng.integers(2, 7)))
    mats = [P.baseline_orthotropic(), P.pagano(), P.isotropic(0.5, 0.3)]
    pool = [float(a) for a in rng.uniform(-1.5, 1.5, size=int(rng.integers(3, 10)))]
    layers = [(mats[int(rng.integers(0, 3))] if rng.uniform() < 0.3 else mats[0],
               pool[int(rng.integers(0, len(pool)))]) for _ in range(m)]
    prob = P.LaminateProblem(
        degree_u=pu, degree_v=pv, degree_t=pt,
        knots_u=random_knots(rng, pu, int(rng.integers(1, 4))),
        knots_v=random_knots(rng, pv, int(rng.integers(1, 4))), knots_t=kt,
        interfaces=ifc, layers=layers, geometry=(float(rng.uniform(0.5, 2)), float(rng.uniform(0.5, 2))),
        direction=(0.0, 0.0, float(rng.uniform(0.05, 0.5))))
    if rng.uniform() < 0.25:
        prob = prob.replace(active_layers=sorted(set(int(x) for x in rng.integers(0, m, size=3))))
    if rng.uniform() < 0.25:
        prob = prob.replace(decompose_angles=True)
    return prob


@pytest.mark.parametrize("min_terms", ["5", "1"])
@pytest.mark.parametrize("seed", range(24))
def test_random_many_angle_laminate_matches_oracle(gpu, oracle, monkeypatch, seed, min_terms):
    """Many-angle laminates against the oracle with the slot form at its
    default threshold and forced for every term count; a function range cut
    inside thickness rows on every third seed."""
    import torch
    monkeypatch.setenv("LAMFAST_SLOTS_MIN_TERMS", min_terms)
    prob = random_many_angle_problem(seed)
    got = gpu.assemble_fast(prob)
    want = oracle.assemble(prob, "fast", want_stats=True)
    assert_csr_match(got.astuple(), want[:3], 1e-12)
    assert got.stats.operator_builds == want[3].operator_builds
    if seed % 3 == 0 and prob.n_t >= 3:
        ns = prob.n_s
        f0, f1 = ns // 2, (prob.n_t - 1) * ns + ns // 3
        plan = gpu.Plan(prob, "fast", 0, f_begin=f0, f_end=f1)
        rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
        cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
        vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
        plan.build_pattern(rp.data_ptr(), cols.data_ptr())
        plan.assemble(vals.data_ptr())
        plan.synchronize()
        trp, tc, tv = want[:3]
        a, e = 3 * f0, 3 * f1
        ref = (trp[a:e + 1] - trp[a], tc[trp[a]:trp[e]], tv[trp[a]:trp[e]])
        assert_csr_match((rp.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy()), ref, 1e-12)
        plan.close()

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

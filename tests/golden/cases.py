"""Small problems whose reference outputs are frozen in tests/golden/.

Shared by make_golden.py (which runs the compiled reference, oracle/_ref) and
the tests (which check the oracle and the GPU path against the fixtures)."""
from paper_1905_05417_b200 import problem as P

HALF_PI = 1.5707963267948966
QUARTER_PI = 0.7853981633974483


def mixed_c0(geom="flat"):
    prob = P.LaminateProblem(
        degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3),
        knots_v=P.uniform_knots(3, 2), knots_t=P.c0_knots(2, 3),
        interfaces=P.equal_interfaces(3),
        layers=[(P.baseline_orthotropic(), 0.0), (P.isotropic(0.5, 0.3), 0.0),
                (P.baseline_orthotropic(), 0.6)])
    if geom == "skewed":
        prob = prob.replace(geometry_kind=1,
                            geometry=(0, 0, 0, 1.2, 0.1, 0.05, -0.1, 0.9, -0.02, 1.0, 1.1, 0.08),
                            direction=(0.03, -0.02, 0.2))
    return prob


def cases():
    """name -> (problem, backends)"""
    return {
        # test_assembly.cpp:129-141 hexahedron: p=1 unit cube, isotropic E=1 nu=0.3
        "hex_p1": (P.cube_problem(1, 1, 1, [(P.isotropic(1.0, 0.3), 0.0)], thickness=1.0),
                   ("standard", "fast", "voigt_free")),
        # test_fast.cpp:310-333 equivalence configs
        "eq_p1": (P.cube_problem(1, 1, 1, [0.0]), ("standard", "fast", "voigt_free")),
        "eq_p2_skewed": (P.cube_problem(2, 2, 1, [0.0, HALF_PI, 0.0], geometry="skewed"),
                         ("standard", "fast", "voigt_free")),
        "eq_p3": (P.cube_problem(3, 2, 1, [0.0, QUARTER_PI, -QUARTER_PI, HALF_PI]),
                  ("standard", "fast", "voigt_free")),
        # test_fast.cpp:354-375 reduced vs long form setup (2 thickness elements)
        "reduced_p2": (P.cube_problem(2, 2, 2, [0.0, HALF_PI, HALF_PI, 0.0], lx=1.3, ly=0.8,
                                      thickness=0.2), ("standard", "fast")),
        # shapes no reference test covers: mixed degrees + C0 thickness knots
        "mixed_c0_flat": (mixed_c0("flat"), ("standard", "fast", "voigt_free")),
        "mixed_c0_skewed": (mixed_c0("skewed"), ("standard", "fast")),
        # masked layers: standard drops fully masked spans
        "masked_c1like": (P.plate(2, 3, 3, [0.0, HALF_PI, HALF_PI, 0.0], thickness=0.1)
                          .replace(active_layers=[1, 2]), ("standard", "fast")),
        # angle decomposition (fast only)
        "decomposed": (P.cube_problem(2, 2, 1, [-1.2, 0.3, 0.9, 1.4], geometry="skewed")
                       .replace(decompose_angles=True), ("fast",)),
    }

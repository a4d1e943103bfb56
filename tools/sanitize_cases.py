"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) over every device kernel family: fast (affine, general), standard,
Voigt-free, decompose_angles, many terms, slabs, operators, verification.  Usage:
  compute-sanitizer --tool racecheck python tools/sanitize_cases.py"""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_05417_b200 as lf
from paper_1905_05417_b200 import problem as P

c1 = P.baseline_config("C1")
skew = P.cube_problem(2, 2, 2, [0.0, 0.9, 0.3], geometry="skewed")
mixed = P.LaminateProblem(
    degree_u=2, degree_v=3, degree_t=2, knots_u=P.uniform_knots(2, 3), knots_v=P.uniform_knots(3, 2),
    knots_t=P.c0_knots(2, 3), interfaces=P.equal_interfaces(3),
    layers=[(P.baseline_orthotropic(), 0.0), (P.isotropic(0.5, 0.3), 0.0), (P.baseline_orthotropic(), 0.6)])
many = P.cube_problem(1, 2, 1, [0.1 * k for k in range(10)])  # 10 terms -> 2 passes
out = []
for prob in (c1, skew, mixed):
    for backend in ("fast", "standard", "voigt_free"):
        out.append(lf.assemble_with(backend, prob).values.sum())
out.append(lf.assemble_fast(c1.replace(decompose_angles=True)).values.sum())
out.append(lf.assemble_fast(many).values.sum())
# general in-plane operators (two-phase)
skew3 = P.cube_problem(3, 3, 1, [0.0, 0.9, 0.3, 1.2], geometry="skewed")
out.append(lf.assemble_fast(skew3).values.sum())
# matrix-free bilinear form (K8)
for prob in (c1, skew, mixed):
    out.append(lf.reference_bilinear(prob, np.ones(prob.dim), np.linspace(0, 1, prob.dim)))
# operator-level entry points (affine + general P, thickness Q, long-form combine)
d = np.diag([1, 1, 1, 0.5, 0.5, 0.5]).astype(float)
for prob in (c1, skew):
    blocks, flags, _ = lf.compute_inplane_operators(prob, d)
    out.append(blocks.sum())
q, occ = lf.compute_thickness_operators(2, skew.knots_t, skew.interfaces, 3)
blocks, flags, _ = lf.compute_inplane_operators(skew, d)
out.append(lf.combine_operators(skew, np.stack([blocks] * len(skew.layers)), flags, q, occ).values.sum())
# slab plan + device verification kernels
import torch
b = lf.slab_bounds(c1, 2, 1)
plan = lf.Plan(c1, "fast", 0, b["t_begin"], b["t_end"])
rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
plan.build_pattern(rp.data_ptr(), cols.data_ptr())
plan.assemble(vals.data_ptr())
plan.synchronize()
st = lf.device_csr_stats(plan.rows, rp.data_ptr(), cols.data_ptr(), vals.data_ptr())
out.append(st["fro_sq"])
plan.close()
# many-term combines (12 terms) on a function range cut inside thickness rows: the slot form
# (default: two terms under any function), the coefficient form, and the slot form with three
# slots (C1 thickness splines: three plies under a function)
many12 = P.plate(2, 6, 5, [(P.baseline_orthotropic(), -1.5 + 0.2 * k) for k in range(12)], thickness=0.2)
many_c1 = P.plate(2, 5, 4, [(P.baseline_orthotropic(), -1.2 + 0.5 * (k % 6)) for k in range(9)], thickness=0.2,
                  thickness_knots=P.uniform_knots(2, 9))
for prob, env, form in ((many12, {}, "slots"), (many12, {"LAMFAST_SLOTS_MIN_TERMS": "1000"}, "coefficient"),
                        (many_c1, {}, "slots")):
    os.environ.update(env)
    plan = lf.Plan(prob, "fast", 0, f_begin=prob.n_s + 5, f_end=4 * prob.n_s - 7)
    for k in env:
        os.environ.pop(k)
    assert plan.combine_form == form, (plan.combine_form, form)
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    out.append(float(vals.sum()))
    plan.close()
# a BASELINE-size plan (C3): the large-slab pattern kernel (16 entries per thread) and the
# 4-term combine with the branch-free bodies
c3 = P.baseline_config("C3")
plan = lf.Plan(c3, "fast", 0)
rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
plan.build_pattern(rp.data_ptr(), cols.data_ptr())
plan.assemble(vals.data_ptr())
plan.synchronize()
out.append(float(vals[:1000].sum()))
plan.close()
print("ok", len(out), float(np.sum(out)))

#!/usr/bin/env python
"""Runs K fast-assembly steps of a BASELINE config on cuda:0 (for ncu / nsight
captures and quick timing).  Prints per-kernel event timing."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1905_05417_b200 as lf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--backend", default="fast")
ap.add_argument("--plies", type=int, default=0)
ap.add_argument("--calibrate", action="store_true")
ap.add_argument("--geometry", default="planar", choices=["planar", "bilinear"])
ap.add_argument("--decompose", action="store_true", help="AssemblyOptions::decompose_angles")
ap.add_argument("--distinct", type=int, default=0,
                help="replace the layup by the orthotropic material at N distinct angles, cycling")
a = ap.parse_args()
if a.calibrate:
    # same-box write-only and copy bandwidth of a buffer the size of C4's values
    n = 1924851600
    buf = torch.empty(n, dtype=torch.float64, device="cuda")
    src = torch.empty(n // 2, dtype=torch.float64, device="cuda")
    dst = torch.empty(n // 2, dtype=torch.float64, device="cuda")
    for name, fn, nbytes in (("fill", lambda: buf.fill_(1.0), n * 8),
                             ("copy", lambda: dst.copy_(src), n * 8)):
        fn()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(10):
            fn()
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / 10
        print(f"calibrate {name}: {nbytes / ms / 1e6:.1f} GB/s ({ms:.3f} ms)")
    del buf, src, dst
    torch.cuda.empty_cache()
prob = lf.baseline_config(a.config, plies=a.plies or None)
if a.geometry == "bilinear":  # non-affine map: general in-plane path (k_inplane_general)
    lx, ly = prob.geometry[0], prob.geometry[1]
    prob = prob.replace(geometry_kind=1, geometry=(0, 0, 0, lx, 0.05 * ly, 0.0, -0.05 * lx, ly, 0.0,
                                                   1.02 * lx, 1.03 * ly, 0.01))
if a.decompose:
    prob = prob.replace(decompose_angles=True)
if a.distinct:
    prob = prob.replace(layers=[(lf.baseline_orthotropic(), -1.5 + 3.0 * (k % a.distinct) / a.distinct)
                                for k in range(len(prob.layers))])
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
plan = lf.Plan(prob, a.backend, 0, stream=s.cuda_stream)
vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
plan.build_pattern(rp.data_ptr(), cols.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
plan.assemble(vals.data_ptr())
torch.cuda.synchronize()
plan.kernel_time(reset=True)
e0.record(s)
for _ in range(a.steps):
    plan.assemble(vals.data_ptr())
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
kms, kn = plan.kernel_time(reset=True)
print(f"{a.config} {a.backend} nnz={plan.nnz} step={ms:.3f} ms combine={kms / max(kn, 1):.3f} ms "
      f"-> {plan.nnz / ms / 1e6:.3e} nnz/s, combine {plan.nnz * 8 / (kms / max(kn, 1)) / 1e6:.1f} GB/s, "
      f"launches/step={plan.launch_count}")

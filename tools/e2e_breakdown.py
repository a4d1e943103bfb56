"""Where the e2e (lf_assemble -> host CSR) time goes: plan creation (host setup
+ table upload), pattern, values, D2H.  python tools/e2e_breakdown.py C4"""
import ctypes
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_1905_05417_b200 as lf
from paper_1905_05417_b200 import abi, problem as P

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
prob = P.baseline_config(name)
lib = abi.library()
c = prob.to_c()
t0 = time.perf_counter()
dim, nnz = ctypes.c_int64(), ctypes.c_int64()
abi.check(lib.lf_pattern_size(ctypes.byref(c), abi.LF_BACKEND_FAST, ctypes.byref(dim), ctypes.byref(nnz)))
t_size = time.perf_counter() - t0
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = lf.Plan(prob, "fast", 0)
    t_plan = time.perf_counter() - t0
    rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
    cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    plan.synchronize()
    t_pat = time.perf_counter() - t0
    t0 = time.perf_counter()
    plan.assemble(vals.data_ptr())
    plan.synchronize()
    t_val = time.perf_counter() - t0
    h = [torch.empty(x.numel(), dtype=x.dtype, pin_memory=True) for x in (rp, cols, vals)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for hx, dx in zip(h, (rp, cols, vals)):
        hx.copy_(dx)
    torch.cuda.synchronize()
    t_d2h = time.perf_counter() - t0
    plan.close()
    del rp, cols, vals, h
print(f"{name}: pattern_size {t_size*1e3:.1f} ms, plan create {t_plan*1e3:.1f} ms, pattern {t_pat*1e3:.1f} ms, "
      f"values {t_val*1e3:.1f} ms, D2H {t_d2h*1e3:.1f} ms")

"""Where do occasional slow one-shot calls (0.5-1.1 s instead of 0.41 s for C4)
spend their time?  Repeats the phases of lf_assemble through the Plan API with
pinned host buffers, timing each: plan create, pattern, values, D2H of
row_ptr, cols, values.   python tools/e2e_phases.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1905_05417_b200 as lf  # noqa: E402

prob = lf.baseline_config("C4")
dim, nnz = lf.pattern_size(prob)
h = (torch.empty(dim + 1, dtype=torch.int64, pin_memory=True), torch.empty(nnz, dtype=torch.int32, pin_memory=True),
     torch.empty(nnz, dtype=torch.float64, pin_memory=True))
d = [torch.empty_like(t, device="cuda") for t in h]
for rep in range(10):
    t = [time.perf_counter()]
    plan = lf.Plan(prob, "fast", 0)
    t.append(time.perf_counter())
    plan.build_pattern(d[0].data_ptr(), d[1].data_ptr())
    plan.synchronize()
    t.append(time.perf_counter())
    plan.assemble(d[2].data_ptr())
    plan.synchronize()
    t.append(time.perf_counter())
    for hx, dx in zip(h, d):
        hx.copy_(dx)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
    plan.close()
    t.append(time.perf_counter())
    ms = [(b - a) * 1e3 for a, b in zip(t, t[1:])]
    print("plan %.1f pattern %.1f values %.1f d2h_rp %.1f d2h_cols %.1f d2h_vals %.1f close %.1f total %.0f ms"
          % (*ms, (t[-1] - t[0]) * 1e3), flush=True)

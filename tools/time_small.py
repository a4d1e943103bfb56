"""Per-step device time of small cube problems vs ply count (acceptance
timing gates).  python tools/time_small.py"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1905_05417_b200 as lf
from paper_1905_05417_b200 import problem as P
for p, e, ms in ((3, 4, (8, 64)), (4, 8, (64,))):
    for m in ms:
        prob = P.cube_problem(p, e, 1, [0.0 if l % 2 == 0 else 0.5 * P.PI for l in range(m)])
        for backend in ("fast", "standard"):
            plan = lf.Plan(prob, backend, 0)
            v = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
            plan.assemble(v.data_ptr()); plan.synchronize()
            t = []
            for _ in range(5):
                t0 = time.perf_counter(); plan.assemble(v.data_ptr()); plan.synchronize(); t.append(time.perf_counter() - t0)
            print(p, e, m, backend, f"{np.median(t)*1e3:.3f} ms", plan.nnz)
            plan.close()

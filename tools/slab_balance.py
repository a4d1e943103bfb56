"""Per-slab device time of an N-way row-slab split, run one slab after the
other on this GPU: the work each rank of an N-GPU run would do (the path has
no exchange step, so an N-GPU step takes the slowest slab's time).  Reports
per-slab ms, nnz and the max/mean imbalance.  This is a load-balance
measurement on one GPU, not a multi-GPU measurement.
    python tools/slab_balance.py --config C4 --parts 8 --scaling weak
    python tools/slab_balance.py --config C5 --parts 8 --scaling strong"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1905_05417_b200 as lf  # noqa: E402
from paper_1905_05417_b200 import problem as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--parts", type=int, default=8)
ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
base = len(P.baseline_config(a.config).layers)
plies = base * a.parts if a.scaling == "weak" else base
prob = P.baseline_config(a.config, plies=plies)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
rows = []
vals = None
for k in range(a.parts):
    b = lf.slab_bounds(prob, a.parts, k)
    plan = lf.Plan(prob, "fast", 0, b["t_begin"], b["t_end"], stream=s.cuda_stream)
    if vals is None or vals.numel() < plan.nnz:
        vals = None
        torch.cuda.empty_cache()
        vals = torch.empty(int(plan.nnz * 1.05), dtype=torch.float64, device="cuda")
    plan.assemble(vals.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.steps):
        plan.assemble(vals.data_ptr())
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    rows.append((k, b["t_begin"], b["t_end"], plan.nnz, ms))
    print(f"slab {k}: t [{b['t_begin']}, {b['t_end']}) nnz {plan.nnz:,} {ms:.3f} ms "
          f"-> {plan.nnz / (ms / 1e3):.3e} nnz/s", flush=True)
    plan.close()
mean = sum(r[4] for r in rows) / len(rows)
mx = max(r[4] for r in rows)
tot = sum(r[3] for r in rows)
print(f"{a.config} {a.scaling} x{a.parts}: total nnz {tot:,}; slab ms mean {mean:.3f} max {mx:.3f} "
      f"(max/mean {mx / mean:.3f}); an {a.parts}-GPU step at the slowest slab: "
      f"{tot / (mx / 1e3):.3e} nnz/s = {tot / mx / (rows[0][3] / rows[0][4]):.2f} x slab 0's rate")

"""lf_assemble (C4, pinned host buffers) timed 5x, then a plain pinned D2H of
the same arrays, in one process: python tools/e2e_ab.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1905_05417_b200 as lf  # noqa: E402

prob = lf.baseline_config("C4")
dim, nnz = lf.pattern_size(prob)
out = (torch.empty(dim + 1, dtype=torch.int64, pin_memory=True), torch.empty(nnz, dtype=torch.int32, pin_memory=True),
       torch.empty(nnz, dtype=torch.float64, pin_memory=True))
np_out = tuple(t.numpy() for t in out)
lf.assemble_with("fast", prob, out=np_out)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    lf.assemble_with("fast", prob, out=np_out)
    ts.append((time.perf_counter() - t0) * 1e3)
srcs = [torch.empty_like(t, device="cuda") for t in out]
ps = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for h, d in zip(out, srcs):
        h.copy_(d)
    torch.cuda.synchronize()
    ps.append((time.perf_counter() - t0) * 1e3)
print(f"lf_assemble ms: {' '.join(f'{t:.0f}' for t in ts)} | plain D2H of the same arrays ms: "
      f"{' '.join(f'{t:.0f}' for t in ps)}")

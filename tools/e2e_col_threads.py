"""lf_assemble (C4, pinned host buffers) with the host column writer on 1..16
threads (LAMFAST_COL_THREADS), 5 calls each, then a plain pinned D2H of the
arrays that cross PCIe: python tools/e2e_col_threads.py"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1905_05417_b200 as lf  # noqa: E402

prob = lf.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
dim, nnz = lf.pattern_size(prob)
out = (torch.empty(dim + 1, dtype=torch.int64, pin_memory=True), torch.empty(nnz, dtype=torch.int32, pin_memory=True),
       torch.empty(nnz, dtype=torch.float64, pin_memory=True))
np_out = tuple(t.numpy() for t in out)
lf.assemble_with("fast", prob, out=np_out)
for rep in range(2):
    for nt in ("default", "2", "3", "4", "6", "8", "12", "16", "24", "32"):
        if nt == "default":
            os.environ.pop("LAMFAST_COL_THREADS", None)
        else:
            os.environ["LAMFAST_COL_THREADS"] = nt
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            lf.assemble_with("fast", prob, out=np_out)
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"col threads {nt:>7}: median {statistics.median(ts):.0f} ms  ({' '.join(f'{t:.0f}' for t in ts)})", flush=True)
srcs = [torch.empty_like(t, device="cuda") for t in (out[0], out[2])]
ps = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for h, d in zip((out[0], out[2]), srcs):
        h.copy_(d)
    torch.cuda.synchronize()
    ps.append((time.perf_counter() - t0) * 1e3)
print(f"plain D2H of row offsets + values ms: {' '.join(f'{t:.0f}' for t in ps)}; host cores {os.cpu_count()}")

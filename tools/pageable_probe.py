"""D2H into pageable vs pinned host memory (the C++ drop-in returns std::vectors,
i.e. pageable memory), and lf_assemble into pageable numpy arrays for C4.
    python tools/pageable_probe.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1905_05417_b200 as lf  # noqa: E402

n = 15_398_812_800 // 8  # C4 values
dev = torch.empty(n, dtype=torch.float64, device="cuda")
for kind in ("pinned", "pageable"):
    host = torch.empty(n, dtype=torch.float64, pin_memory=(kind == "pinned"))
    host.zero_()
    best = 0.0
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host.copy_(dev)
        torch.cuda.synchronize()
        best = max(best, n * 8 / (time.perf_counter() - t0) / 1e9)
    print(f"{kind:9s} D2H 15.4 GB: {best:.1f} GB/s")
    del host
del dev
prob = lf.baseline_config("C4")
dim, nnz = lf.pattern_size(prob)
out = (np.empty(dim + 1, np.int64), np.empty(nnz, np.int32), np.empty(nnz))
for a in out:
    a.fill(0)
for rep in range(2):
    t0 = time.perf_counter()
    lf.assemble_with("fast", prob, out=out)
    print(f"lf_assemble C4 into pageable numpy: {(time.perf_counter() - t0) * 1e3:.0f} ms")

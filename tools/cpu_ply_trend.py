"""Reference CPU fast-assembly rate (oracle/_ref, the unmodified reference
sources) against the ply count of a BASELINE config family: shows whether a
few-ply sample stands for the full laminate's nnz/s.
  python tools/cpu_ply_trend.py C4 2 9 32"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.checkers import Reference  # noqa: E402
from paper_1905_05417_b200 import problem as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
plies = [int(x) for x in sys.argv[2:]] or [2, 9, 32]
ref = Reference()
threads = os.cpu_count() or 1
print(f"# {cfg} family, reference assembleFast, threads={threads}, one warm-up + one timed call per size")
for m in plies:
    prob = P.baseline_config(cfg, plies=m)
    nnz = P.sizes(prob)["nnz"]
    ref.assemble(P.baseline_config(cfg, plies=1), "fast", threads)
    t0 = time.perf_counter()
    ref.assemble(prob, "fast", threads)
    dt = time.perf_counter() - t0
    print(f"{cfg} plies={m:4d} nnz={nnz:12d} {dt:8.2f} s  {nnz / dt:.3e} nnz/s", flush=True)

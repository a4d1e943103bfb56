"""C5's 203 GB CSR streamed through lf_assemble_stream (bench.measure_stream_e2e)
against the number of host threads writing each chunk's columns
(LAMFAST_COL_THREADS): python tools/c5_stream_threads.py [threads ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1905_05417_b200 import problem as P  # noqa: E402

prob = P.baseline_config("C5")
total = P.sizes(prob)["nnz"]
for nt in sys.argv[1:] or ["default"]:
    if nt == "default":
        os.environ.pop("LAMFAST_COL_THREADS", None)
    else:
        os.environ["LAMFAST_COL_THREADS"] = nt
    r = bench.measure_stream_e2e(prob, 0, total)
    print(f"col threads {nt}: {r['ms']:.0f} ms (warm-up {r['warmup_ms']:.0f} ms), {r['value']:.3e} nnz/s, "
          f"{r['d2h_gbs']:.1f} GB/s over PCIe", flush=True)

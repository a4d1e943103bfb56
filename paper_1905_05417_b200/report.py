"""Benchmark report in the reference's format, extended with throughput.

Mirrors the reference's bench report (bench.hpp:128-168, bench.cpp:245-299):
one record per (backend, config) with the reference's columns
``backend,p,elements,m,m_bar,time_s,nnz,rel_diff,qpoints`` followed by the
B200 columns ``elements_y,nnz_per_s,hbm_frac``.  Times are device times of
one full assembly (CUDA events, median of the repetitions) with the problem
resident; rel_diff is frobeniusRelDiff against the standard backend of the
same config, computed on the device (lf_csr_diff_sq).

  python -m paper_1905_05417_b200.report --configs C1 C2 --backends standard fast --format csv
"""
from __future__ import annotations

import argparse
import ctypes
import io
import json
import os
import statistics
import sys
from dataclasses import asdict, dataclass, field
from typing import List, Optional

from . import abi

CSV_HEADER = "backend,p,elements,m,m_bar,time_s,nnz,rel_diff,qpoints"
EXTRA_COLUMNS = "elements_y,nnz_per_s,hbm_frac"


@dataclass
class Record:
    backend: str
    p: int
    elements: int
    m: int
    m_bar: int
    time_s: float
    nnz: int
    rel_diff: Optional[float]
    qpoints: int
    elements_y: int = 0
    nnz_per_s: float = 0.0
    hbm_frac: float = 0.0


@dataclass
class Report:
    records: List[Record] = field(default_factory=list)
    failures: List[str] = field(default_factory=list)
    threads: int = 1


def emit_csv(report: Report, out=None) -> str:
    buf = io.StringIO()
    buf.write(CSV_HEADER + "," + EXTRA_COLUMNS + "\n")
    for r in report.records:
        rel = "" if r.rel_diff is None else repr(r.rel_diff)
        buf.write(f"{r.backend},{r.p},{r.elements},{r.m},{r.m_bar},{r.time_s!r},{r.nnz},{rel},"
                  f"{r.qpoints},{r.elements_y},{r.nnz_per_s!r},{r.hbm_frac!r}\n")
    text = buf.getvalue()
    if out is not None:
        out.write(text)
    return text


def emit_json(report: Report) -> str:
    return json.dumps({"records": [asdict(r) for r in report.records], "failures": report.failures,
                       "threads": report.threads}, indent=1)


def parse_json(text: str) -> Report:
    doc = json.loads(text)
    return Report([Record(**r) for r in doc["records"]], list(doc["failures"]), int(doc["threads"]))


def _hbm_gbs() -> float:
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def run(configs, backends, device: int = 0, repetitions: int = 5) -> Report:
    """Device-resident sweep over BASELINE configs (names) x backends."""
    import torch
    from .assembler import Plan
    from .problem import baseline_config

    torch.cuda.set_device(device)
    stream = torch.cuda.Stream()  # the plans run on this stream; events must too
    torch.cuda.set_stream(stream)
    lib = abi.library()
    hbm = _hbm_gbs()
    report = Report()
    for name in configs:
        prob = baseline_config(name)
        resident = {}
        for backend in backends:
            try:
                plan = Plan(prob, backend, device, stream=stream.cuda_stream)
                rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
                cols = torch.empty(max(1, plan.nnz), dtype=torch.int32, device="cuda")
                vals = torch.empty(max(1, plan.nnz), dtype=torch.float64, device="cuda")
                plan.build_pattern(rp.data_ptr(), cols.data_ptr())
                plan.assemble(vals.data_ptr())  # warm-up
                torch.cuda.synchronize()
                times = []
                for _ in range(repetitions):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    plan.assemble(vals.data_ptr())
                    e1.record(stream)
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1) / 1e3)
                t = statistics.median(times)
                st = plan.stats()
                plan.close()
                resident[backend] = (rp, cols, vals)
                report.records.append(Record(
                    backend=backend, p=prob.degree_u, elements=len(prob.knots_u) - 2 * prob.degree_u - 1,
                    m=prob.n_layers, m_bar=prob.distinct_configs(), time_s=t, nnz=plan.nnz,
                    rel_diff=None, qpoints=int(st.qpoint_visits),
                    elements_y=len(prob.knots_v) - 2 * prob.degree_v - 1, nnz_per_s=plan.nnz / t,
                    hbm_frac=plan.nnz * 8 / t / (hbm * 1e9)))
            except Exception as exc:  # recorded, the sweep continues (bench.cpp:189-191)
                report.failures.append(f"{name} backend={backend}: {exc}")
        if "standard" in resident:
            rs = resident["standard"]
            fro_s = ctypes.c_double()
            abi.check(lib.lf_csr_frobenius_sq(prob.dim, ctypes.c_void_p(rs[0].data_ptr()),
                                              ctypes.c_void_p(rs[2].data_ptr()), None,
                                              ctypes.byref(fro_s)))
            for rec in report.records:
                if rec.backend == "standard" or rec.backend not in resident or rec.m != prob.n_layers:
                    continue
                ra = resident[rec.backend]
                d2, fro_a = ctypes.c_double(), ctypes.c_double()
                abi.check(lib.lf_csr_diff_sq(prob.dim, *(ctypes.c_void_p(x.data_ptr()) for x in ra),
                                             *(ctypes.c_void_p(x.data_ptr()) for x in rs), None,
                                             ctypes.byref(d2)))
                abi.check(lib.lf_csr_frobenius_sq(prob.dim, ctypes.c_void_p(ra[0].data_ptr()),
                                                  ctypes.c_void_p(ra[2].data_ptr()), None,
                                                  ctypes.byref(fro_a)))
                den = max(fro_a.value, fro_s.value) ** 0.5
                rec.rel_diff = 0.0 if den == 0 else d2.value ** 0.5 / den
        del resident
        torch.cuda.empty_cache()
    report.records.sort(key=lambda r: (r.backend, r.p, r.elements, r.m))
    return report


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["C1", "C2"])
    ap.add_argument("--backends", nargs="+", default=["standard", "fast"])
    ap.add_argument("--repetitions", type=int, default=5)
    ap.add_argument("--format", choices=["csv", "json"], default="csv")
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    rep = run(a.configs, a.backends, a.device, a.repetitions)
    sys.stdout.write(emit_csv(rep) if a.format == "csv" else emit_json(rep) + "\n")


if __name__ == "__main__":
    main()

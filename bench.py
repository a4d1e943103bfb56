#!/usr/bin/env python
"""Benchmark: assembled FP64 CSR stiffness nnz/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

One step = one complete fast assembly (assembleFast: basis evaluation,
thickness integrals, in-plane operators, combination into the FP64 CSR
values) of the workload, inputs resident in HBM.  Workload at N=1: BASELINE
config C4 (128x64 elements, p=2, 128 plies, 1.92e9 nnz, 23 GB CSR) -- the
largest BASELINE config that fits one B200 with its pattern (C5 is 203 GB).
With N ranks (torchrun) the path partitions into row slabs,
one per GPU, cut at function boundaries and balanced by nnz, no collective on
the data path.  Default --scaling weak: the laminate of the config family
grows with N (N x 128 plies for C4) and each rank assembles one slab of it,
i.e. one C4's worth of rows per GPU; --scaling strong splits the fixed config
across the N GPUs instead.

Also in the line (each its own timed region, never inside the headline one):
  c5            BASELINE C5 (the scaling case, 1.69e10 nnz) split over the N
                ranks (strong scaling): per-rank device time, max over ranks,
                balance, roofline; at N=1 also its streamed e2e (203 GB
                through lf_assemble_stream into pinned host staging);
  e2e_dropin    the C++ drop-in's assembleFast (std::vector result in
                pageable memory) timed by build/dropin_e2e.

Reported beside the device number:
  e2e           the same metric through the C-ABI one-shot call lf_assemble
                (the drop-in for assembleFast) with pinned host buffers: H2D
                of the problem tables + the whole CSR (row offsets, columns,
                values) D2H inside the timed region;
  roofline      8 B/nnz FP64 value stores of the combine kernel (K4) against
                the measured HBM copy bandwidth (MEASURED_PEAKS.json);
  cpu_baseline  the reference's own fast assembler (compiled from its
                unmodified sources, oracle/_ref) on a bounded sample of the
                same workload family, all host threads;
  standard      side measurement: the standard full-3D quadrature assembly
                (assembleStandard, the path the fast one replaces) on the
                same workload on this GPU, and the reference's own
                assembleStandard on a 1-ply sample on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-plies", type=int, default=0)
    ap.add_argument("--no-standard", action="store_true",
                    help="skip the standard-assembly (cross-check path) side measurement")
    ap.add_argument("--verify-gather", action="store_true",
                    help="N>1 over NCCL: also gather the full CSR to rank 0 when it fits and check it there")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: N x the config's plies, one slab per GPU; strong: the config split N ways")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the multi-rank path on fewer GPUs than ranks")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 strong-scaling sub-measurement")
    ap.add_argument("--no-dropin", action="store_true", help="skip the C++ drop-in e2e timing")
    ap.add_argument("--no-oracle-check", action="store_true",
                    help="N>1: skip the per-rank oracle comparison of one sampled thickness row")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU fast assembler (oracle/_ref),
    all host threads, on a bounded sample of the workload family."""
    if rank != 0:
        return
    import resource
    from oracle.checkers import Reference
    from paper_1905_05417_b200 import problem as P
    if not Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref_lamfast.so not built"}))
        return
    ref = Reference()
    threads = os.cpu_count() or 1
    plies = choose_sample_plies(ref, args, threads, budget_s=150.0)
    prob = P.baseline_config(args.config, plies=plies)
    nnz = P.sizes(prob)["nnz"]
    full_plies = len(P.baseline_config(args.config).layers)
    for _ in range(args.warmup):
        ref.assemble(prob, "fast", threads)
    times = []
    ru0 = resource.getrusage(resource.RUSAGE_SELF)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.assemble(prob, "fast", threads)
        times.append(time.perf_counter() - t0)
    ru1 = resource.getrusage(resource.RUSAGE_SELF)
    cpu_s = (ru1.ru_utime - ru0.ru_utime) + (ru1.ru_stime - ru0.ru_stime)
    wall = sum(times)
    sec = wall / len(times)
    value = nnz / sec
    sample = (f"{args.config} family with {plies} plies instead of {full_plies} (same elements, degree, "
              f"materials); {nnz} nnz per step")
    line = {
        "impl": "reference", "metric": "assembled stiffness nnz/s (FP64 CSR)", "value": value,
        "unit": "nnz/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "backend": "fast", "sample_plies": plies,
                   "nnz_per_step": nnz, "same_config": plies == full_plies,
                   "same_config_reason": None if plies == full_plies else
                   (f"the full {args.config} takes minutes per step on the host (reference ~8e6 nnz/s vs "
                    f"{P.sizes(P.baseline_config(args.config))['nnz']:.3g} nnz), so each step is the "
                    f"first {plies} plies of the same laminate; the reference's rate is flat in the "
                    f"ply count (profiles/r2_cpu_ply_trend.txt)")},
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads, "kind": "reference",
                         "sample": sample, "threads_requested": threads,
                         "effective_parallelism": cpu_s / wall if wall > 0 else None,
                         "note": "AssemblyOptions.threads = all host threads; the reference's "
                                 "SparseMatrixBuilder merge and stable_sort run on one thread, so the "
                                 "measured CPU-time/wall ratio is the effective parallelism"},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def choose_sample_plies(ref, args, threads, budget_s):
    """Largest ply count of the config family whose reference run keeps
    (warmup + steps) within budget_s; calibrated with a 1-ply run."""
    from paper_1905_05417_b200 import problem as P
    if args.cpu_sample_plies:
        return args.cpu_sample_plies
    probe = P.baseline_config(args.config, plies=1)
    t0 = time.perf_counter()
    ref.assemble(probe, "fast", threads)
    dt = time.perf_counter() - t0
    rate = P.sizes(probe)["nnz"] / max(dt, 1e-6)
    per_step = budget_s / max(1, args.steps + args.warmup)
    full = len(P.baseline_config(args.config).layers)
    best = 1
    for m in range(1, full + 1):
        if P.sizes(P.baseline_config(args.config, plies=m))["nnz"] / rate <= per_step:
            best = m
        else:
            break
    return best


def cpu_baseline(args):
    """Reference fast path (oracle/_ref) on a bounded sample, ~10-30 s."""
    from oracle.checkers import Reference
    from paper_1905_05417_b200 import problem as P
    if not Reference.available():
        return None
    ref = Reference()
    threads = os.cpu_count() or 1
    a = argparse.Namespace(**vars(args))
    a.steps, a.warmup = 1, 0
    plies = choose_sample_plies(ref, a, threads, budget_s=20.0)
    prob = P.baseline_config(args.config, plies=plies)
    nnz = P.sizes(prob)["nnz"]
    import resource
    ru0 = resource.getrusage(resource.RUSAGE_SELF)
    t0 = time.perf_counter()
    ref.assemble(prob, "fast", threads)
    dt = time.perf_counter() - t0
    ru1 = resource.getrusage(resource.RUSAGE_SELF)
    cpu_s = (ru1.ru_utime - ru0.ru_utime) + (ru1.ru_stime - ru0.ru_stime)
    return {"value": nnz / dt, "unit": "nnz/s", "cores": threads, "kind": "reference",
            "effective_parallelism": cpu_s / dt if dt > 0 else None,
            "sample": f"{args.config} family with {plies} plies ({nnz} nnz), one assembleFast, "
                      f"reference sources compiled with the Eigen subset, threads={threads} "
                      f"(AssemblyOptions.threads; its merge and stable_sort are serial)"}


def device_step_time(plans, vals_ptrs, steps, warmup, stream, world, dist_backend):
    """Event-timed steps of the given plans (one step = every plan once),
    barrier + synchronize on both sides, max over ranks.  Returns (ms per
    step, combine ms per step, combine launches, launches per step)."""
    import torch
    import torch.distributed as dist

    def step():
        for p, v in zip(plans, vals_ptrs):
            p.assemble(v)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    for p in plans:
        p.kernel_time(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    k_ms = k_n = 0
    for p in plans:
        a, b = p.kernel_time(reset=True)
        k_ms += a
        k_n += b
    local = (ms / steps, k_ms / steps)
    t = torch.tensor(list(local), dtype=torch.float64)
    per_rank = [local]
    if world > 1:
        tc = t.cuda() if dist_backend == "nccl" else t
        gathered = [torch.empty_like(tc) for _ in range(world)]
        dist.all_gather(gathered, tc)
        per_rank = [tuple(float(x) for x in g.cpu()) for g in gathered]
    return {"ms_per_step": max(r[0] for r in per_rank), "combine_ms_per_step": k_ms / steps,
            "combine_launches": k_n, "launches_per_step": sum(p.launch_count for p in plans),
            "per_rank_ms": [r[0] for r in per_rank], "local_ms": local[0]}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    if world > 1:
        # NCCL's own log (stderr) records the communicator size per rank
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # the per-rank oracle check shares the host cores
        os.environ.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 1) // world)))
    import torch
    import torch.distributed as dist
    import paper_1905_05417_b200 as lf
    from paper_1905_05417_b200 import problem as P

    device = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(args.dist_backend)
    base_plies = len(P.baseline_config(args.config).layers)
    plies = base_plies * world if args.scaling == "weak" else base_plies
    prob = P.baseline_config(args.config, plies=plies)
    sz = P.sizes(prob)
    # this rank's slab: functions [f_begin, f_end), cut inside thickness rows,
    # balanced by nnz to within one function
    bounds = (lf.slab_bounds_functions(prob, world, rank) if world > 1 else
              {"f_begin": 0, "f_end": prob.n_s * prob.n_t, "row_begin": 0, "nnz_begin": 0})
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    # pattern + values resident when both fit; else values only, in as few
    # sequential sub-slab passes as the values need
    free, _ = torch.cuda.mem_get_info()
    full = lf.Plan(prob, "fast", device, stream=stream.cuda_stream, f_begin=bounds["f_begin"],
                   f_end=bounds["f_end"])
    with_pattern = full.nnz * 12 + full.rows * 8 <= int(0.85 * free)
    passes = 1 if with_pattern else max(1, -(-full.nnz * 8 // int(0.9 * free)))
    if passes == 1:
        plans = [full]
    else:
        full.close()
        f0, f1 = bounds["f_begin"], bounds["f_end"]
        cuts = [f0 + ((f1 - f0) * k) // passes for k in range(passes + 1)]
        plans = [lf.Plan(prob, "fast", device, stream=stream.cuda_stream, f_begin=cuts[k], f_end=cuts[k + 1])
                 for k in range(passes)]
    vals = torch.empty(max(p.nnz for p in plans), dtype=torch.float64, device="cuda")
    rp = cols = None
    if with_pattern:
        plan = plans[0]
        rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
        cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
        plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    torch.cuda.synchronize()
    # the precomputed CSR pattern (K5), reported separately (outside the timed
    # region): 4 B per column + 8 B per row offset
    pattern = None
    if with_pattern:
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for _ in range(3):
            plan.build_pattern(rp.data_ptr(), cols.data_ptr())
        p1.record(stream)
        torch.cuda.synchronize()
        pms = p0.elapsed_time(p1) / 3
        pbytes = plan.nnz * 4 + (plan.rows + 1) * 8
        pattern = {"ms": pms, "bytes": pbytes, "gbs": pbytes / (pms / 1e3) / 1e9,
                   "kernels": "k_pattern_rows + k_pattern_cols"}

    sampler = ClockSampler(device)
    sampler.start()
    timing = device_step_time(plans, [vals.data_ptr()] * len(plans), args.steps, args.warmup, stream, world,
                              args.dist_backend)
    clocks = sampler.stop()
    ms_per_step = timing["ms_per_step"]
    launches = timing["launches_per_step"] * args.steps
    rank_nnz = sum(p.nnz for p in plans)
    # combine kernel: average duration of one launch over all sub-slabs -> bytes/s
    k_avg_ms = timing["combine_ms_per_step"] * args.steps / max(timing["combine_launches"], 1)
    k_bytes = rank_nnz * 8 / len(plans)
    total_nnz = sz["nnz"]
    value = total_nnz / (ms_per_step / 1e3)

    # verification of the resident matrix (outside the timed region)
    verify = {}
    if world == 1 and with_pattern:
        st = lf.device_csr_stats(plans[0].rows, rp.data_ptr(), cols.data_ptr(), vals.data_ptr(),
                                 stream.cuda_stream)
        verify = {"fro_norm": st["fro_sq"] ** 0.5, "symmetry_rel": (st["sym_sq"] / st["fro_sq"]) ** 0.5,
                  "symmetry_rel_closed_form": (plans[0].symmetry_sq(vals.data_ptr()) / st["fro_sq"]) ** 0.5}
    elif world > 1 and with_pattern:
        from paper_1905_05417_b200 import distributed as D
        s = D.slab_summary(rp, cols, vals[:plans[0].nnz], bounds["row_begin"], bounds["nnz_begin"])
        if not args.no_oracle_check:  # verification leg, outside the timed region
            from oracle.checkers import slab_oracle_delta
            s = D.with_field(s, "oracle_rel_dk", slab_oracle_delta(prob, bounds["f_begin"], bounds["f_end"], rp,
                                                                    cols, vals[:plans[0].nnz]))
        parts = D.gather_summaries(s.cuda() if args.dist_backend == "nccl" else s)
        tot = D.combine_summaries(parts)
        verify = {"fro_norm": tot["fro_sq"] ** 0.5, "nnz_gathered": int(tot["nnz"]),
                  "rows_gathered": int(tot["rows"]), "pattern_hash": tot["pattern_hash"],
                  "pattern_hash_closed_form_ok": int(tot["nnz"]) == total_nnz and int(tot["rows"]) == sz["dim"],
                  "oracle_max_rel_dk_per_rank": [float(p[D.FIELD_INDEX["oracle_rel_dk"]]) for p in parts]
                  if not args.no_oracle_check else None,
                  "nccl_ranks": world}
        # full-slab gather to rank 0 over NCCL where the whole K fits there
        fits = torch.tensor([1.0 if (sz["nnz"] * 12 + sz["dim"] * 8) * 2 <= 0.8 * torch.cuda.mem_get_info()[0]
                             else 0.0], dtype=torch.float64, device="cuda")
        if args.dist_backend == "nccl" and args.verify_gather:
            dist.all_reduce(fits, op=dist.ReduceOp.MIN)
            if float(fits[0]) > 0:
                full_csr = D.gather_csr(rp, cols, vals[:plans[0].nnz], dst=0)
                if rank == 0:
                    g_rp, g_cols, g_vals = full_csr
                    st = lf.device_csr_stats(sz["dim"], g_rp.data_ptr(), g_cols.data_ptr(), g_vals.data_ptr(),
                                             stream.cuda_stream)
                    verify["full_gather"] = {"fro_norm": st["fro_sq"] ** 0.5,
                                             "symmetry_rel": (st["sym_sq"] / st["fro_sq"]) ** 0.5,
                                             "rows": int(g_rp.numel() - 1), "nnz": int(g_cols.numel())}
                del full_csr
                torch.cuda.empty_cache()

    hbm, peak_src = peaks()
    if pattern:
        pattern["frac"] = pattern["gbs"] / hbm
    achieved = k_bytes / (k_avg_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None,
                "kernel": "k_combine (K4)", "bytes_per_launch": k_bytes,
                "kernel_ms": k_avg_ms, "peak_source": peak_src,
                "step_frac": value * 8 / (world * hbm * 1e9)}
    # ncu DRAM traffic is attached only to the exact workload it was captured on
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        try:
            with open(traffic_file) as f:
                tj = json.load(f).get(args.config)
            if tj and world == 1 and passes == 1 and plies == base_plies:
                roofline["traffic"] = tj["dram_bytes_per_launch"]
                roofline["traffic_source"] = tj["source"]
            elif tj:
                roofline["traffic_note"] = (f"ncu traffic is from the 1-GPU {args.config} capture; this "
                                            f"line's per-rank workload differs, so traffic is null")
        except Exception:
            pass
    del rp, cols, vals
    for p in plans:
        p.close()
    torch.cuda.empty_cache()
    # context for the write-only kernel: a plain write-only fill of a buffer of
    # the same size on this GPU (torch fill_, best of 3, CUDA events)
    try:
        fbuf = torch.empty(int(k_bytes // 8), dtype=torch.float64, device="cuda")
        fbuf.fill_(0.0)
        best = 0.0
        for _ in range(3):
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            fbuf.fill_(1.0)
            f1.record()
            torch.cuda.synchronize()
            best = max(best, fbuf.numel() * 8 / (f0.elapsed_time(f1) / 1e3) / 1e9)
        roofline["write_fill_gbs"] = best
        roofline["frac_of_write_fill"] = achieved / best
        del fbuf
        torch.cuda.empty_cache()
    except Exception:
        pass

    e2e = None
    if not args.no_e2e:
        try:
            if world == 1:
                e2e = measure_e2e(args, prob, device, total_nnz)
            else:
                e2e = measure_e2e_slab(args, prob, device, rank, world, bounds, total_nnz)
        except Exception as exc:  # e.g. pinned host memory limits: reported, the device line stands
            e2e = {"value": None, "unit": "nnz/s", "error": f"{type(exc).__name__}: {exc}"[:300]}
    lf.release_memory(device)

    e2e_dropin = None
    if world == 1 and not args.no_dropin:
        e2e_dropin = measure_e2e_dropin(args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args)
        except Exception as exc:  # reported, not fatal
            cpu = {"error": str(exc)}

    standard = None
    if world == 1 and with_pattern and not args.no_standard:
        try:
            standard = measure_standard(args, prob, device, stream)
            standard["gpu_fast_over_standard"] = standard["gpu"]["ms_per_step"] / ms_per_step
        except Exception as exc:  # reported, not fatal
            standard = {"error": str(exc)}

    many = None
    if world == 1 and with_pattern and not args.no_standard:
        try:
            many = measure_many_terms(args, prob, device, stream, hbm)
        except Exception as exc:  # reported, not fatal
            many = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    c5 = None
    if not args.no_c5 and args.config != "C5":
        try:
            c5 = measure_c5(args, device, rank, world, stream, hbm)
        except Exception as exc:  # reported, not fatal
            c5 = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if rank == 0:
        line = {
            "metric": "assembled stiffness nnz/s (FP64 CSR)", "value": value, "unit": "nnz/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config if world == 1 or args.scaling == "strong"
                       else f"{args.config} family, {plies} plies ({world} x {base_plies}), one slab per GPU",
                       "backend": "fast", "nnz": total_nnz,
                       "dofs": sz["dim"], "plies": len(prob.layers),
                       "distinct_materials": prob.distinct_configs(),
                       "l2": "output > L2 (values %.1f GB vs 126 MB L2); no flush needed"
                             % (total_nnz * 8 / 1e9),
                       "parallelism": f"row-slab x{world}", "slab_cuts": "function boundaries, nnz-balanced",
                       "slab_passes_per_gpu": passes},
            "roofline": roofline, "e2e": e2e, "e2e_dropin": e2e_dropin, "cpu_baseline": cpu,
            "gpu_launches": launches, "clocks": clocks, "verify": verify, "standard": standard,
            "pattern": pattern, "per_rank_ms": timing["per_rank_ms"], "c5": c5, "many_terms": many,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def measure_c5(args, device, rank, world, stream, hbm):
    """BASELINE C5 (the scaling case: 192x192 p=3, 128 random-angle plies,
    1.69e10 nnz) split over the N ranks by function-level nnz-balanced slabs
    (strong scaling): per-rank device time of the whole hot path, max over
    ranks; at N=1 also its streamed e2e.  Pattern resident where it fits,
    else values only (1 GPU: 135 GB of values)."""
    import torch
    import paper_1905_05417_b200 as lf
    from paper_1905_05417_b200 import problem as P
    prob = P.baseline_config("C5")
    total = P.sizes(prob)["nnz"]
    b = lf.slab_bounds_functions(prob, world, rank) if world > 1 else {"f_begin": 0, "f_end": prob.n_s * prob.n_t}
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    free //= max(1, -(-world // max(1, torch.cuda.device_count())))  # ranks sharing a GPU (code-path runs)
    plan = lf.Plan(prob, "fast", device, stream=stream.cuda_stream, f_begin=b["f_begin"], f_end=b["f_end"])
    nnz = plan.nnz
    with_pattern = nnz * 12 + plan.rows * 8 <= int(0.85 * free)
    fits = with_pattern or nnz * 8 <= int(0.9 * free)
    if world > 1:  # every rank takes the same branch (the timing below has collectives)
        import torch.distributed as dist
        flags = torch.tensor([1.0 if fits else 0.0, 1.0 if with_pattern else 0.0], dtype=torch.float64)
        if args.dist_backend == "nccl":
            flags = flags.cuda()
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        fits, with_pattern = bool(flags[0] > 0), bool(flags[1] > 0)
    if not fits:
        plan.close()
        return {"error": f"the C5 slab's values ({nnz * 8 / 1e9:.0f} GB on rank {rank}) do not fit on every rank"}
    vals = torch.empty(nnz, dtype=torch.float64, device="cuda")
    rp = cols = None
    if with_pattern:
        rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
        cols = torch.empty(nnz, dtype=torch.int32, device="cuda")
        plan.build_pattern(rp.data_ptr(), cols.data_ptr())
    steps, warmup = max(3, min(args.steps, 10)), 2
    sampler = ClockSampler(device)
    sampler.start()
    t = device_step_time([plan], [vals.data_ptr()], steps, warmup, stream, world, args.dist_backend)
    clocks = sampler.stop()
    k_ms = t["combine_ms_per_step"]
    out = {"workload": "C5 (192x192, p=3, 128 plies, 4 materials), row slabs at function boundaries",
           "scaling": "strong", "nnz": total, "steps": steps, "warmup": warmup,
           "ms_per_step": t["ms_per_step"], "value": total / (t["ms_per_step"] / 1e3), "unit": "nnz/s",
           "per_rank_ms": t["per_rank_ms"],
           "balance_max_over_mean": max(t["per_rank_ms"]) / (sum(t["per_rank_ms"]) / len(t["per_rank_ms"])),
           "rank0_nnz": nnz, "pattern_resident": with_pattern, "clocks": clocks,
           "roofline": {"bound": "hbm", "kernel": "k_combine (K4)", "achieved": nnz * 8 / (k_ms / 1e3) / 1e9,
                        "peak": hbm, "frac": nnz * 8 / (k_ms / 1e3) / 1e9 / hbm, "unit": "GB/s",
                        "step_frac": total * 8 / (t["ms_per_step"] / 1e3) / (world * hbm * 1e9)}}
    if with_pattern:
        st = lf.device_csr_stats(plan.rows, rp.data_ptr(), cols.data_ptr(), vals.data_ptr(), stream.cuda_stream)
        out["rank0_fro_norm"] = st["fro_sq"] ** 0.5
    plan.close()
    del vals, rp, cols
    torch.cuda.empty_cache()
    if world == 1 and not args.no_e2e:
        out["e2e_stream"] = measure_stream_e2e(prob, device, total)
    lf.release_memory(device)
    return out


def measure_stream_e2e(prob, device, total_nnz):
    """C5's 203 GB CSR (more than HBM and than this host's RAM) streamed
    through lf_assemble_stream: every chunk computed on the device and copied
    into pinned host staging, handed to a sink that sums its values (so the
    bytes are really read on the host).  One warm-up call, one timed."""
    import ctypes
    import numpy as np
    from paper_1905_05417_b200 import abi
    lib = abi.library()
    c = prob.to_c()
    acc = {"sum": 0.0, "chunks": 0, "bytes": 0, "pcie": 0}

    def sink(_u, row_begin, rows, nnz_begin, nnz, rp, cols, vals):
        acc["chunks"] += 1
        acc["bytes"] += (rows + 1) * 8 + nnz * 12
        acc["pcie"] += (rows + 1) * 8 + nnz * (8 if host_columns() else 12)
        acc["sum"] += float(np.ctypeslib.as_array(vals, shape=(nnz,))[::4096].sum()) if nnz else 0.0
        return 0

    fn = abi.CHUNK_SINK(sink)
    st = abi.Stats()
    times = []
    for _ in range(2):
        acc.update(sum=0.0, chunks=0, bytes=0, pcie=0)
        t0 = time.perf_counter()
        abi.check(lib.lf_assemble_stream(ctypes.byref(c), abi.LF_BACKEND_FAST, device, 0,
                                         ctypes.cast(fn, ctypes.c_void_p), None, ctypes.byref(st)))
        times.append(time.perf_counter() - t0)
    sec = times[-1]
    return {"value": total_nnz / sec, "unit": "nnz/s", "ms": sec * 1e3, "chunks": acc["chunks"],
            "csr_bytes": acc["bytes"], "d2h_bytes": acc["pcie"], "d2h_gbs": acc["pcie"] / sec / 1e9,
            "warmup_ms": times[0] * 1e3,
            "columns": "written on the host per chunk into the staging slot while its values cross PCIe"
                       if host_columns() else "device pattern copied over PCIe",
            "call": "lf_assemble_stream(LF_BACKEND_FAST) -> pinned host staging -> sink (sampled sum)"}


def measure_e2e_dropin(args):
    """The C++ drop-in as a reference-API caller uses it: lamfast::assembleFast
    returning a StiffnessMatrix of std::vectors (pageable memory), timed by
    build/dropin_e2e (3 calls after a warm-up)."""
    exe = os.path.join(ROOT, "build", "dropin_e2e")
    if not os.path.exists(exe):
        return {"unavailable": "build/dropin_e2e not built"}
    try:
        r = subprocess.run([exe, args.config if args.config in ("C2", "C3", "C4") else "C4", "3"],
                           capture_output=True, text=True, timeout=600)
        out = json.loads(r.stdout.strip().splitlines()[-1])
        out["unit"] = "nnz/s"
        out["call"] = "lamfast::assembleFast(setup) -> StiffnessMatrix (std::vector, pageable)"
        return out
    except Exception as exc:
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def measure_standard(args, prob, device, stream):
    """Side measurement (not the headline): the standard full-3D quadrature
    assembly (assembleStandard, the path the fast one replaces) on the same
    workload -- device nnz/s on this GPU (k_standard, event-timed, values in
    the same precomputed CSR) and the reference's own assembleStandard
    (oracle/_ref, all host threads) on a bounded sample of the family."""
    import torch
    import paper_1905_05417_b200 as lf
    from paper_1905_05417_b200 import problem as P
    out = {}
    plan = lf.Plan(prob, "standard", device, stream=stream.cuda_stream)
    vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    plan.assemble(vals.data_ptr())  # warm-up
    torch.cuda.synchronize()
    steps = 2
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        plan.assemble(vals.data_ptr())
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    out["gpu"] = {"value": plan.nnz / (ms / 1e3), "unit": "nnz/s", "ms_per_step": ms, "steps": steps,
                  "launches_per_step": plan.launch_count, "workload": args.config}
    plan.close()
    del vals
    torch.cuda.empty_cache()
    if not args.no_cpu_baseline:
        from oracle.checkers import Reference
        if Reference.available():
            ref = Reference()
            threads = os.cpu_count() or 1
            sample = P.baseline_config(args.config, plies=1)
            nnz = P.sizes(sample)["nnz"]
            t0 = time.perf_counter()
            ref.assemble(sample, "standard", threads)
            dt = time.perf_counter() - t0
            out["cpu_baseline"] = {
                "value": nnz / dt, "unit": "nnz/s", "cores": threads, "kind": "reference",
                "sample": f"{args.config} family with 1 ply ({nnz} nnz), one assembleStandard, "
                          f"reference sources compiled with the Eigen subset, threads={threads}"}
    return out


def measure_many_terms(args, prob, device, stream, hbm):
    """Side measurement: the same workload with many operator terms, one
    launch whatever the term count: AssemblyOptions.decompose_angles (five
    basis terms per material; on this affine map they are summed per distinct
    ply configuration before the combine, so the per-term kernel runs with the
    direct form's three terms) and the orthotropic ply at 16 distinct angles
    (two terms under any function: the slot form, k_combine_slots).
    Device time per step (CUDA events) and the combine's HBM fraction, values
    in the same precomputed pattern."""
    import torch
    import paper_1905_05417_b200 as lf
    orth = lf.baseline_orthotropic()
    cases = {"decompose_angles": prob.replace(decompose_angles=True),
             "16_distinct_angles": prob.replace(layers=[(orth, -1.5 + 3.0 * (k % 16) / 16)
                                                        for k in range(len(prob.layers))])}
    out = {}
    for name, pr in cases.items():
        plan = lf.Plan(pr, "fast", device, stream=stream.cuda_stream)
        vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
        t = device_step_time([plan], [vals.data_ptr()], max(3, min(args.steps, 10)), 2, stream, 1, "nccl")
        k_ms = t["combine_ms_per_step"]
        out[name] = {"ms_per_step": t["ms_per_step"], "value": plan.nnz / (t["ms_per_step"] / 1e3),
                     "unit": "nnz/s", "operator_builds": plan.stats().operator_builds,
                     "launches_per_step": plan.launch_count,
                     "form": plan.combine_form,
                     "combine_ms": k_ms, "combine_frac_of_hbm": plan.nnz * 8 / (k_ms / 1e3) / 1e9 / hbm}
        plan.close()
        del vals
        torch.cuda.empty_cache()
    return out


def host_columns() -> bool:
    """One-shot calls write the CSR columns on the host (lf_pattern_columns)
    unless LAMFAST_HOST_COLS=0; then only row offsets and values cross PCIe."""
    return os.environ.get("LAMFAST_HOST_COLS", "1") != "0"


def measure_e2e(args, prob, device, total_nnz):
    """lf_assemble (drop-in for assembleFast) with pinned host buffers.  The
    columns are written by host threads while row offsets and values cross
    PCIe (default); the same call with the device pattern copied over PCIe
    (LAMFAST_HOST_COLS=0) is timed beside it."""
    import torch
    from paper_1905_05417_b200 import abi
    lib = abi.library()
    c = prob.to_c()
    dim = prob.dim
    rp = torch.empty(dim + 1, dtype=torch.int64, pin_memory=True)
    cols = torch.empty(total_nnz, dtype=torch.int32, pin_memory=True)
    vals = torch.empty(total_nnz, dtype=torch.float64, pin_memory=True)
    st = abi.Stats()

    def once():
        abi.check(lib.lf_assemble(ctypes.byref(c), abi.LF_BACKEND_FAST, device, rp.data_ptr(),
                                  cols.data_ptr(), vals.data_ptr(), ctypes.byref(st)))

    def timed(n):
        once()  # warm-up (allocator pool, module load)
        per = []
        t0 = time.perf_counter()
        for _ in range(n):
            t1 = time.perf_counter()
            once()
            per.append(time.perf_counter() - t1)
        return (time.perf_counter() - t0) / n, per

    hc = host_columns()
    sec, per = timed(max(1, args.e2e_steps))
    alt = None
    if hc:  # the device-pattern variant of the same call, for comparison
        os.environ["LAMFAST_HOST_COLS"] = "0"
        try:
            alt_sec, _ = timed(2)
            alt = {"ms_per_step": alt_sec * 1e3, "value": total_nnz / alt_sec,
                   "d2h_bytes_per_step": rp.numel() * 8 + total_nnz * 12}
        finally:
            os.environ.pop("LAMFAST_HOST_COLS", None)
    h2d = sum(a.nbytes for a in prob._keep if hasattr(a, "nbytes"))
    d2h = rp.numel() * 8 + total_nnz * (8 if hc else 12)
    # the e2e roofline: a plain pinned D2H of the arrays that cross PCIe
    # (device tensors of the CSR's sizes into the same pinned buffers), after
    # the timed region, best of 2
    dev = f"cuda:{device}"
    hosts = (rp, vals) if hc else (rp, cols, vals)
    srcs = [torch.empty_like(h, device=dev) for h in hosts]
    best = 0.0
    for _ in range(2):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for h, dsrc in zip(hosts, srcs):
            h.copy_(dsrc)
        torch.cuda.synchronize()
        best = max(best, d2h / (time.perf_counter() - t1) / 1e9)
    del rp, cols, vals, srcs, hosts
    return {"value": total_nnz / sec, "unit": "nnz/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": sec * 1e3, "steps": len(per),
            "call": "lf_assemble(LF_BACKEND_FAST) -> host CSR (row_ptr, cols, values)",
            "columns": "written on the host (closed form, lf_pattern_columns) while row offsets and values "
                       "cross PCIe" if hc else "device pattern copied over PCIe",
            "ms_median": statistics.median(per) * 1e3,
            "d2h_gbs_measured": best, "d2h_probe": "plain pinned D2H of the arrays that cross PCIe, best of 2",
            "pcie_frac": (d2h / sec / 1e9) / best if best else None,
            "device_columns": alt}


def measure_e2e_slab(args, prob, device, rank, world, bounds, total_nnz):
    """Per-rank e2e of the slab path through the C-ABI one-shot call
    lf_assemble_slab (setup + table H2D, pattern, values, D2H of the slab
    CSR into pinned host buffers, the pattern read back while the values are
    computed); max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_1905_05417_b200 as lf
    probe = lf.Plan(prob, "fast", device, f_begin=bounds["f_begin"], f_end=bounds["f_end"])
    rows, nnz = probe.rows, probe.nnz
    probe.close()
    # every rank must get its buffers before any enters a collective
    err = ""
    try:
        out = (torch.empty(rows + 1, dtype=torch.int64, pin_memory=True),
               torch.empty(nnz, dtype=torch.int32, pin_memory=True),
               torch.empty(nnz, dtype=torch.float64, pin_memory=True))
    except Exception as exc:
        err = f"rank {rank}: {type(exc).__name__}: {exc}"[:300]
    ok = torch.tensor([0.0 if err else 1.0], dtype=torch.float64)
    if args.dist_backend == "nccl":
        ok = ok.cuda()
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if float(ok[0]) < 1.0:
        return {"value": None, "unit": "nnz/s", "error": err or "buffer allocation failed on another rank"}

    def once():
        lf.assemble_range(prob, bounds["f_begin"], bounds["f_end"], "fast", device, out=out)

    once()
    dist.barrier()
    n = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(n):
        once()
    dt = torch.tensor([(time.perf_counter() - t0) / n], dtype=torch.float64)
    if args.dist_backend == "nccl":
        dt = dt.cuda()
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    sec = float(dt[0])
    h2d = sum(a.nbytes for a in prob._keep if hasattr(a, "nbytes"))
    d2h = torch.tensor([float((rows + 1) * 8 + nnz * (8 if host_columns() else 12))], dtype=torch.float64)
    if args.dist_backend == "nccl":
        d2h = d2h.cuda()
    dist.all_reduce(d2h)
    return {"value": total_nnz / sec, "unit": "nnz/s", "h2d_bytes_per_step": int(h2d) * world,
            "d2h_bytes_per_step": int(d2h[0]), "ms_per_step": sec * 1e3, "steps": n,
            "call": "per rank: lf_assemble_range (setup + table H2D, pattern, values, slab CSR D2H)"}


if __name__ == "__main__":
    main()

"""Row-slab sharding across GPUs.

The assembly has no exchange step: rank r of N assembles the contiguous row
slab ``slab_bounds_functions(prob, N, r)`` (cut at function boundaries, i.e.
inside thickness rows, balanced by nnz to within one function) into its own
HBM, with row offsets rebased to 0 and global column indices.  Collectives (NCCL over NVLink on GPUs, gloo on CPU) are used
only for verification -- gathering per-slab summaries -- never inside the
timed assembly.
"""
from __future__ import annotations

import os
from typing import Dict, List

from .assembler import slab_bounds, slab_bounds_functions
from .problem import LaminateProblem

SUMMARY_FIELDS = ("rows", "nnz", "fro_sq", "checksum", "max_abs", "pattern_hash", "oracle_rel_dk")
FIELD_INDEX = {k: i for i, k in enumerate(SUMMARY_FIELDS)}
HASH_P = (1 << 31) - 1  # pattern hashes are sums mod this prime: exact in float64 across ranks


def env_rank():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def slab_for_rank(prob: LaminateProblem, rank: int, world: int, backend: str = "fast") -> Dict[str, int]:
    """This rank's row slab: functions [f_begin, f_end), nnz-balanced (cuts
    inside thickness rows)."""
    return slab_bounds_functions(prob, world, rank, backend)


def _mix(x):
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic, logical
    shifts), reduced to [0, HASH_P)."""
    import torch

    def shr(v, s):
        return (v >> s) & ((1 << (64 - s)) - 1)
    x = x ^ shr(x, 30)
    x = x * -4658895280553007687  # 0xbf58476d1ce4e5b9 as int64
    x = x ^ shr(x, 27)
    x = x * -7723592293110705685  # 0x94d049bb133111eb as int64
    x = x ^ shr(x, 31)
    return torch.remainder(shr(x, 1), HASH_P)


def pattern_hash(row_ptr, cols, row_begin: int = 0, nnz_begin: int = 0, chunk: int = 1 << 27) -> int:
    """Additive hash of a slab's CSR pattern in global coordinates: every
    (global entry position, column) and every (global row, global row
    offset) contributes mix(.) mod HASH_P, so the slabs' hashes sum (mod
    HASH_P) to the full matrix's.  Runs on the tensors' device, in chunks."""
    import torch
    rp = torch.as_tensor(row_ptr).to(torch.int64)
    c = torch.as_tensor(cols)
    nnz = int(rp[-1] - rp[0])
    dev = c.device
    h = 0
    for lo in range(0, nnz, chunk):
        hi = min(nnz, lo + chunk)
        pos = torch.arange(lo + nnz_begin, hi + nnz_begin, dtype=torch.int64, device=dev)
        h += int(_mix((pos << 32) | c[lo:hi].to(torch.int64)).sum())
    rows = len(rp) - 1
    for lo in range(0, rows, chunk):
        hi = min(rows, lo + chunk)
        r = torch.arange(lo + row_begin, hi + row_begin, dtype=torch.int64, device=rp.device)
        h += int(_mix((r << 40) ^ (rp[lo:hi] - rp[0] + nnz_begin) ^ (1 << 62)).sum())
    return h % HASH_P


def slab_summary(row_ptr, cols, values, row_begin: int = 0, nnz_begin: int = 0):
    """Summary of one slab CSR (torch tensors on any device, or numpy):
    rows, nnz, sum of squares, a position-weighted checksum, max |v|, and
    the additive pattern hash (global coordinates: pass the slab's first
    global row and nnz offset).  The checksum weights each value by its
    global column, so a value stored in the wrong column changes it."""
    import torch
    rp = torch.as_tensor(row_ptr)
    c = torch.as_tensor(cols)
    v = torch.as_tensor(values).to(torch.float64)
    nnz = int(rp[-1] - rp[0])
    v = v[:nnz]
    c = c[:nnz]
    w = (c.to(torch.int64) % 97 + 1).to(torch.float64)
    ph = pattern_hash(rp, c, row_begin, nnz_begin)
    return torch.tensor([float(len(rp) - 1), float(nnz), float((v * v).sum()),
                         float((v * w).sum()), float(v.abs().max()) if nnz else 0.0, float(ph), -1.0],
                        dtype=torch.float64)


def with_field(summary, name: str, value: float):
    """A copy of a slab summary with one field set (e.g. the oracle_rel_dk a
    verification leg computed for this rank's slab)."""
    s = summary.clone()
    s[FIELD_INDEX[name]] = float(value)
    return s


def gather_summaries(summary, group=None) -> List:
    """all_gather of the per-rank summaries (verification only)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = summary.device
    if dist.get_backend(group) == "nccl" and dev.type != "cuda":
        summary = summary.cuda()
    out = [torch.empty_like(summary) for _ in range(world)]
    dist.all_gather(out, summary, group=group)
    return [o.to(dev) for o in out]


def combine_summaries(parts) -> Dict[str, float]:
    tot = {k: 0.0 for k in SUMMARY_FIELDS}
    for p in parts:
        for i, k in enumerate(SUMMARY_FIELDS):
            tot[k] = max(tot[k], float(p[i])) if k in ("max_abs", "oracle_rel_dk") else tot[k] + float(p[i])
    tot["pattern_hash"] = int(tot["pattern_hash"]) % HASH_P
    return tot


def gather_csr(row_ptr, cols, values, dst: int = 0, group=None):
    """Full-slab gather for verification (only where the whole
    K fits one device -- C1..C4, up to 23 GB): every rank sends its slab CSR
    (row offsets rebased to 0, global columns) to rank `dst` with
    point-to-point send/recv (NCCL over NVLink on GPUs, gloo on CPU); `dst`
    returns the whole matrix (row_ptr, cols, values) in rank order, the
    others None.  Never on the timed path."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    rp = torch.as_tensor(row_ptr)
    c = torch.as_tensor(cols)
    v = torch.as_tensor(values)
    nnz = int(rp[-1] - rp[0])
    dev = c.device
    nccl = dist.get_backend(group) == "nccl"
    comm_dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    sizes = torch.tensor([len(rp) - 1, nnz], dtype=torch.int64, device=comm_dev)
    all_sizes = [torch.empty_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [(int(s[0]), int(s[1])) for s in all_sizes]
    rp_local = (rp[:-1] - rp[0]).to(comm_dev)
    c_local = c[:nnz].to(comm_dev)
    v_local = v[:nnz].to(comm_dev)
    if rank != dst:
        for t in (rp_local, c_local, v_local):
            dist.send(t.contiguous(), dst, group=group)
        return None
    parts = []
    for r in range(world):
        rows_r, nnz_r = all_sizes[r]
        if r == dst:
            parts.append((rp_local, c_local, v_local))
            continue
        bufs = (torch.empty(rows_r, dtype=rp_local.dtype, device=comm_dev),
                torch.empty(nnz_r, dtype=c_local.dtype, device=comm_dev),
                torch.empty(nnz_r, dtype=v_local.dtype, device=comm_dev))
        for t in bufs:
            dist.recv(t, r, group=group)
        parts.append(bufs)
    offs, rps = 0, []
    for (prp, pc, _), (_, nnz_r) in zip(parts, all_sizes):
        rps.append(prp + offs)
        offs += nnz_r
    rps.append(torch.tensor([offs], dtype=rp_local.dtype, device=comm_dev))
    return (torch.cat(rps).to(dev), torch.cat([p[1] for p in parts]).to(dev),
            torch.cat([p[2] for p in parts]).to(dev))

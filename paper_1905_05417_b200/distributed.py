"""Row-slab sharding across GPUs.

The assembly has no exchange step: rank r of N assembles the contiguous row
slab ``slab_bounds(prob, N, r)`` (cut at thickness-function boundaries,
balanced by nnz) into its own HBM, with row offsets rebased to 0 and global
column indices.  Collectives (NCCL over NVLink on GPUs, gloo on CPU) are used
only for verification -- gathering per-slab summaries -- never inside the
timed assembly.
"""
from __future__ import annotations

import os
from typing import Dict, List

from .assembler import slab_bounds
from .problem import LaminateProblem

SUMMARY_FIELDS = ("rows", "nnz", "fro_sq", "checksum", "max_abs")


def env_rank():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def slab_for_rank(prob: LaminateProblem, rank: int, world: int, backend: str = "fast") -> Dict[str, int]:
    return slab_bounds(prob, world, rank, backend)


def slab_summary(row_ptr, cols, values):
    """Summary of one slab CSR (torch tensors on any device, or numpy):
    rows, nnz, sum of squares, a position-weighted checksum, max |v|.
    The checksum weights each value by its global column, so a value stored
    in the wrong column changes it."""
    import torch
    rp = torch.as_tensor(row_ptr)
    c = torch.as_tensor(cols)
    v = torch.as_tensor(values).to(torch.float64)
    nnz = int(rp[-1] - rp[0])
    v = v[:nnz]
    c = c[:nnz]
    w = (c.to(torch.int64) % 97 + 1).to(torch.float64)
    return torch.tensor([float(len(rp) - 1), float(nnz), float((v * v).sum()),
                         float((v * w).sum()), float(v.abs().max()) if nnz else 0.0],
                        dtype=torch.float64)


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
            tot[k] = max(tot[k], float(p[i])) if k == "max_abs" else tot[k] + float(p[i])
    return tot

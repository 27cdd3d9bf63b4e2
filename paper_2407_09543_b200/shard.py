"""Multi-GPU partitioning of the NTBC hot path.

Every BC word depends only on the model and its block coordinates, so the path shards with no
data-path exchange: block-row ranges of one material (latency view) or whole materials of a batch
(throughput view).  The only collective is the final gather of packed BC words to rank 0, which
BASELINE.json's north star counts in the timing.  These helpers are backend-agnostic (NCCL on GPU
tensors, gloo on CPU tensors for the tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def row_shards(block_rows: int, world: int):
    """Contiguous, balanced [begin, end) block-row ranges, one per rank (sizes differ by <= 1)."""
    if world < 1 or block_rows < 1:
        raise ValueError("need world >= 1 and block_rows >= 1")
    base, extra = divmod(block_rows, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < extra else 0)
        out.append((b, e))
        b = e
    return out


def material_shards(n_materials: int, world: int):
    """Materials assigned round-robin-contiguously: rank r decodes materials [lo_r, hi_r)."""
    return row_shards(n_materials, world)


def gather_rows(local: torch.Tensor, shards, rank: int, world: int, group=None):
    """Gather per-rank row shards of a [n_tex, rows_r, BW] int64 tensor into the full
    [n_tex, sum(rows_r), BW] tensor on rank 0 (returns None on other ranks).

    Shards may differ in size by one row, so each rank pads to the largest shard before a
    fixed-size gather (NCCL gather needs equal sizes) and rank 0 trims while assembling."""
    n_tex, _, bw = local.shape
    max_rows = max(e - b for b, e in shards)
    pad = local.new_zeros((n_tex, max_rows, bw))
    pad[:, :local.shape[1]] = local
    if world == 1:
        return pad[:, :shards[0][1] - shards[0][0]].clone()
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, bufs, dst=0, group=group)
    if rank != 0:
        return None
    return torch.cat([bufs[r][:, :e - b] for r, (b, e) in enumerate(shards)], dim=1)


def gather_materials(local: torch.Tensor, rank: int, world: int, group=None):
    """Gather one equally-shaped [n_tex, BH, BW] material per rank to rank 0 (list in rank order)."""
    if world == 1:
        return [local]
    bufs = [torch.empty_like(local) for _ in range(world)] if rank == 0 else None
    dist.gather(local, bufs, dst=0, group=group)
    return bufs if rank == 0 else None

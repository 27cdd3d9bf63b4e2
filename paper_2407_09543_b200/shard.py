"""Multi-GPU partitioning of the NTBC hot path.

Every BC word depends only on the model and its block coordinates, so the path shards with no
data-path exchange: block-row ranges of one material (latency view) or whole materials of a batch
(throughput view).  The only collective is the final gather of packed BC words to rank 0, which
BASELINE.json's north star counts in the timing.  Two implementations:
  * PeerGather (default on GPUs): the gather is fused into the decode -- every rank's fused kernel
    stores its BC words straight into rank 0's buffer through a CUDA-IPC mapping (NVLink), unit by
    unit while later units are computed; a one-element all-reduce then marks completion;
  * gather_rows / gather_materials: a separate collective (dist.gather) after the decode -- NCCL on
    GPU tensors, gloo on CPU tensors for the tests.
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


class _PeerBuffer:
    """Rank 0 allocates an int64 device buffer of `shape` and exports it (ntbc_peer_export); the handle is
    broadcast with the process group; every other rank maps it (ntbc_peer_open).  `base` is the buffer's
    address in this rank's address space.  The ranks agree on success (an all-reduce of the outcome), so
    they fall back together when IPC or peer access is unavailable."""

    def __init__(self, shape, rank: int, world: int, device: torch.device, group=None):
        from . import ntbc   # CUDA only; the CPU helpers above do not need the library
        self.rank, self.world, self.group, self._opened = rank, world, group, None
        self.buf, self.base, self.error = None, None, None
        handle = None
        if rank == 0:
            try:
                self.buf = torch.empty(shape, dtype=torch.int64, device=device)
                handle = ntbc.peer_export(self.buf)
            except Exception as e:   # e.g. an allocator without IPC support
                self.error = f"export: {e}"
        obj = [handle]
        dist.broadcast_object_list(obj, src=0, group=group)
        if rank == 0:
            self.base = self.buf.data_ptr() if handle is not None else None
        elif obj[0] is not None:
            try:
                self.base = self._opened = ntbc.peer_open(obj[0], device.index)
            except Exception as e:   # no peer access between these GPUs
                self.error = f"open: {e}"
        ok = torch.tensor([1 if self.base is not None else 0], dtype=torch.int32,
                          device=device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        self.ok = bool(ok.item())
        self._flag = torch.zeros(1, dtype=torch.int32, device=device)

    def complete(self):
        """All ranks' decodes (issued before this call on the current stream) have landed in rank 0's buffer
        once this all-reduce completes; the current stream waits for it (NCCL).  With a CPU backend (gloo,
        the single-GPU functional test) the host synchronises the device and then joins a barrier."""
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)

    def close(self):
        if self._opened is not None:
            from . import ntbc
            torch.cuda.synchronize()
            ntbc.peer_close(self._opened)
            self._opened = None


class PeerGather(_PeerBuffer):
    """Fused gather of a batch of equally-shaped materials into rank 0's [n_materials, n_tex, BH, BW] buffer
    (throughput view; BASELINE config 5: 64 materials sharded 64/G per rank).  Rank r owns the contiguous
    materials `material_shards(n_materials, world)[r]` and decodes material g straight into its slice
    (ntbc.decode_material(..., out_ptrs=self.ptrs_of(g))); `complete()` is the only exchange on the timed
    path, after which rank 0's buffer holds all materials (the writes are system-scope fenced by the fused
    kernel).  n_materials defaults to one per rank; `ptrs` = the pointers of this rank's first material."""

    def __init__(self, n_tex: int, bh: int, bw: int, rank: int, world: int, device: torch.device, group=None,
                 n_materials: int | None = None):
        n_materials = world if n_materials is None else n_materials
        super().__init__((n_materials, n_tex, bh, bw), rank, world, device, group)
        self.n_tex, self.plane = n_tex, bh * bw * 8
        self.lo, self.hi = material_shards(n_materials, world)[rank]
        self.ptrs = self.ptrs_of(self.lo) if self.ok and self.hi > self.lo else None

    def ptrs_of(self, g: int):
        """Device pointers (this rank's address space) of material g's texture planes in rank 0's buffer."""
        return [self.base + (g * self.n_tex + k) * self.plane for k in range(self.n_tex)]


class PeerRows(_PeerBuffer):
    """One material split by block rows over the ranks (latency view): rank r decodes the rows
    row_shards(BH, world)[r] straight into those rows of rank 0's [n_tex, BH, BW] buffer
    (ntbc.decode_material(..., row_begin=self.r0, row_end=self.r1, out_ptrs=self.ptrs)).  With an odd
    BW the row offsets are only 8-B aligned; the kernel then writes one 8-byte word per block."""

    def __init__(self, n_tex: int, bh: int, bw: int, rank: int, world: int, device: torch.device, group=None):
        super().__init__((n_tex, bh, bw), rank, world, device, group)
        self.r0, self.r1 = row_shards(bh, world)[rank]
        plane = bh * bw * 8
        self.ptrs = [self.base + k * plane + self.r0 * bw * 8 for k in range(n_tex)] if self.ok else None

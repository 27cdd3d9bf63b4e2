"""N>1 host logic on CPU (-m "not gpu"): world_size-2 gloo process group over 127.0.0.1.

Each rank produces the BC words of its block-row shard (here with the oracle, standing in for the
per-GPU decode, which test_gpu_parity.test_row_shards_union_equals_full covers on the device), the
product's gather helper assembles them on rank 0, and the result must equal the single-process
decode byte for byte (SURVEY §8.e equivalence)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_09543_b200.shard import gather_materials, gather_rows, material_shards, row_shards


def test_row_shards_cover_exactly():
    for rows in (1, 7, 64, 1024, 1025):
        for world in (1, 2, 3, 4, 8):
            sh = row_shards(rows, world)
            assert len(sh) == world and sh[0][0] == 0 and sh[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            sizes = [e - b for b, e in sh]
            assert max(sizes) - min(sizes) <= 1
    assert material_shards(64, 8) == [(8 * i, 8 * i + 8) for i in range(8)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, W, H, result):
    import oracle
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blob = synth.model_blob(1)
        om = oracle.Model(blob)
        sh = row_shards(H // 4, world)
        b, e = sh[rank]
        local = torch.from_numpy(om.decode_material(W, H, b, e).astype(np.int64).view(np.int64))
        full = gather_rows(local, sh, rank, world)
        mats = gather_materials(torch.full((2, 3, 4), rank, dtype=torch.int64), rank, world)
        if rank == 0:
            result["rows"] = full.numpy().copy()
            result["mats"] = [m.numpy().copy() for m in mats]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_gather_equals_single_process(world):
    import oracle
    import synth
    W, H = 64, 52                      # 13 block rows: uneven shards (7 + 6)
    mgr = mp.get_context("spawn").Manager()
    result = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), W, H, result), nprocs=world, join=True,
                       start_method="spawn")
    ref = oracle.Model(synth.model_blob(1)).decode_material(W, H)
    assert np.array_equal(result["rows"].view(np.uint64), ref)
    for r, m in enumerate(result["mats"]):
        assert np.all(m == r)


def _worker_batch(rank, world, port, n_mat, result):
    """BASELINE config 5's host logic at world 2 on CPU: materials material_shards(n_mat, world)[rank] decoded
    per rank (the oracle standing in for the GPU decode), gathered to rank 0 one material per rank per call
    (bench.py's NCCL-gather fallback), assembled in global material order."""
    import oracle
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, H = 32, 16
        lo, hi = material_shards(n_mat, world)[rank]
        batch = {}
        for i, g in enumerate(range(lo, hi)):
            words = oracle.Model(synth.model_blob(1, material=g)).decode_material(W, H)
            got = gather_materials(torch.from_numpy(words.astype(np.int64).view(np.int64)), rank, world)
            if rank == 0:
                for r, t in enumerate(got):
                    batch[material_shards(n_mat, world)[r][0] + i] = t.numpy().copy()
        if rank == 0:
            result["batch"] = [batch[g] for g in range(n_mat)]
    finally:
        dist.destroy_process_group()


def test_gloo_material_batch_equals_single_process():
    import oracle
    import synth
    n_mat, world = 4, 2
    mgr = mp.get_context("spawn").Manager()
    result = mgr.dict()
    mp.start_processes(_worker_batch, args=(world, _free_port(), n_mat, result), nprocs=world, join=True,
                       start_method="spawn")
    for g, words in enumerate(result["batch"]):
        ref = oracle.Model(synth.model_blob(1, material=g)).decode_material(32, 16)
        assert np.array_equal(words.view(np.uint64), ref), g

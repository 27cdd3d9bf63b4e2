"""The fused peer-memory gather (ntbc_peer_export / ntbc_peer_open, shard.PeerGather).

Functional test on ONE GPU: two processes (gloo process group for the host coordination) both use
cuda:0; rank 1 maps rank 0's buffer through CUDA IPC and its fused kernel stores its material's BC
words straight into rank 0's slice.  The two kernels never wait on each other (the only coupling is a
host barrier after each process synchronised its device), so this is safe on one GPU; it checks the
plumbing and the addressing, not NVLink bandwidth (that needs the driver's multi-GPU run)."""
import os
import socket
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu

CFG = 2   # 1024^2, 2 BC1 + 1 BC4: a few ms per decode


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2407_09543_b200 import ntbc
    from paper_2407_09543_b200.shard import PeerGather

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    W, H, _ = synth.config_shape(CFG)
    model = ntbc.Model(synth.model_blob(CFG, material=rank), 0)
    pg = PeerGather(model.n_tex, H // 4, W // 4, rank, world, dev)
    ntbc.decode_material([model], W, H, out_ptrs=pg.ptrs)
    pg.complete()
    if rank == 0:
        for r in range(world):   # reference: each material decoded locally into ordinary tensors
            m = ntbc.Model(synth.model_blob(CFG, material=r), 0)
            ref = torch.stack(ntbc.decode_material([m], W, H))
            torch.cuda.synchronize()
            np.save(os.path.join(outdir, f"eq{r}.npy"), np.array([bool(torch.equal(pg.buf[r], ref))]))
    dist.barrier()
    pg.close()
    dist.barrier()
    dist.destroy_process_group()


def test_peer_gather_two_processes_one_gpu(tmp_path):
    import numpy as np
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert bool(np.load(tmp_path / f"eq{r}.npy")[0]), f"rank {r}'s material differs in rank 0's buffer"


def _worker_batch(rank, world, port, outdir):
    """C5-style batch (4 materials, 2 per rank, each decoded into its slice of rank 0's buffer) and the
    latency view (one material split by block rows, BW odd so shard offsets are only 8-B aligned)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2407_09543_b200 import ntbc
    from paper_2407_09543_b200.shard import PeerGather, PeerRows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    W, H = 4 * 251, 4 * 37                      # BW = 251 (odd), BH = 37 (uneven row shards)
    n_mat = 4
    tex = ntbc.Model(synth.model_blob(CFG, material=0), 0).n_tex
    pg = PeerGather(tex, H // 4, W // 4, rank, world, dev, n_materials=n_mat)
    for g in range(pg.lo, pg.hi):
        m = ntbc.Model(synth.model_blob(CFG, material=10 + g), 0)
        ntbc.decode_material([m], W, H, out_ptrs=pg.ptrs_of(g))
    pg.complete()
    pr = PeerRows(tex, H // 4, W // 4, rank, world, dev)
    m0 = ntbc.Model(synth.model_blob(CFG, material=99), 0)
    ntbc.decode_material([m0], W, H, row_begin=pr.r0, row_end=pr.r1, out_ptrs=pr.ptrs)
    pr.complete()
    if rank == 0:
        ok = []
        for g in range(n_mat):
            ref = torch.stack(ntbc.decode_material([ntbc.Model(synth.model_blob(CFG, material=10 + g), 0)], W, H))
            torch.cuda.synchronize()
            ok.append(bool(torch.equal(pg.buf[g], ref)))
        ref = torch.stack(ntbc.decode_material([m0], W, H))
        torch.cuda.synchronize()
        ok.append(bool(torch.equal(pr.buf, ref)))
        np.save(os.path.join(outdir, "batch.npy"), np.array(ok))
    dist.barrier()
    pg.close()
    pr.close()
    dist.barrier()
    dist.destroy_process_group()


def test_peer_gather_batch_and_row_split_two_processes(tmp_path):
    import numpy as np
    import torch.multiprocessing as mp

    mp.spawn(_worker_batch, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    ok = np.load(tmp_path / "batch.npy")
    assert ok.all(), ok


def test_peer_handle_offset_and_errors():
    import torch

    from paper_2407_09543_b200 import ntbc
    t = torch.zeros(1024, dtype=torch.int64, device="cuda")
    h0, h1 = ntbc.peer_export(t), ntbc.peer_export(t[128:])
    assert len(h0) == len(h1) == ntbc.PEER_HANDLE_BYTES
    assert h0[:64] == h1[:64]                                  # same allocation, same IPC handle
    off = lambda h: int.from_bytes(h[64:72], "little")       # noqa: E731
    assert off(h1) - off(h0) == 128 * 8                       # the offset inside the allocation travels along
    with pytest.raises(ntbc.NtbcError):
        ntbc.peer_close(12345)                                 # not a pointer returned by peer_open
    with pytest.raises(ValueError):
        ntbc.peer_open(b"short", 0)

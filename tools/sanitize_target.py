"""compute-sanitizer target: every kernel family of libntbc.so once on the
C1 and C2 shapes -- prep (grid dequant + prefix build), fused decode (NTBC and naive, dump modes, the
conservative pair in one launch, a row shard with 8-B aligned outputs), pack, BC decode, reference
encoder, both training steps (with QAT), the tcgen05 summation probe.  Results are checked against the
oracle where cheap, so a sanitizer-clean run is also a correct one.

usage: compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_target.py [cfgs...]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2407_09543_b200 import ntbc  # noqa: E402

DEV = "cuda:0"


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def main(cfgs):
    for cfg in cfgs:
        W, H, _ = synth.config_shape(cfg)
        blob = synth.model_blob(cfg)
        m = ntbc.Model(blob)
        outs = ntbc.decode_material([m], W, H)
        ep, col = ntbc.debug_mlp(m, W, H, 0, min(H // 4, 8))
        ntbc.debug_features(m, W, H, 0, 2)
        r0, r1 = 1, min(H // 4, 6)                                 # a shard with an odd row offset
        part = torch.zeros((m.n_tex, (r1 - r0) * (W // 4) + 2), dtype=torch.int64, device=DEV)
        ntbc.decode_material([m], W, H, row_begin=r0, row_end=r1,
                             out_ptrs=[part[k].data_ptr() + 8 for k in range(m.n_tex)])   # 8-B aligned planes
        ref = oracle.Model(blob).decode_material(W, H, 0, min(H // 4, 8))
        for k in range(m.n_tex):
            assert np.array_equal(u64(outs[k])[:ref.shape[1]], ref[k]), (cfg, k)
        fmts = m.fmts
        g = ntbc.pack(fmts, ep, col, W, 4 * min(H // 4, 8))
        for k in range(m.n_tex):
            assert np.array_equal(u64(g[k]), ref[k]), ("pack", cfg, k)
            ntbc.decode_bc(outs[k], fmts[k], W, H)
        print(f"C{cfg}: decode / dump / shard / pack / decode_bc ok", flush=True)
    # naive model and the conservative pair (one launch, CTAs partitioned by model)
    W, H, _ = synth.config_shape(8)
    ntbc.decode_material([ntbc.Model(synth.model_blob(8))], W, H)
    rgb = synth.serialize(synth.random_model(synth.ModelSpec([synth.BC1, synth.BC1], block_levels=4, texel_levels=5), 5))
    sc = synth.serialize(synth.random_model(synth.ModelSpec([synth.BC4] * 4, block_levels=4, texel_levels=5), 6))
    pair = ntbc.decode_material([ntbc.Model(rgb), ntbc.Model(sc)], 256, 64)
    ref = list(oracle.Model(rgb).decode_material(256, 64)) + list(oracle.Model(sc).decode_material(256, 64))
    for k in range(6):
        assert np.array_equal(u64(pair[k]), ref[k]), ("pair", k)
    # reference encoder, both formats
    for fmt, ch in ((1, 3), (4, 1)):
        tex = torch.from_numpy(synth.texture(128, 64, ch, seed=fmt)).to(DEV)
        ntbc.encode_bc(tex, fmt, 128, 64, 2)
    # training steps (colour + endpoint, QAT on), small batches
    rng = np.random.default_rng(0)
    fmts = [synth.BC1, synth.BC4]
    for qat in (False, True):
        n = ntbc.train_param_count(fmts, 64, 4, 8)
        p = torch.from_numpy(rng.uniform(-0.5, 0.5, n).astype(np.float32)).to(DEV)
        g, am, av = (torch.zeros(n, device=DEV) for _ in range(3))
        B = 256
        xy = torch.from_numpy(np.stack([rng.integers(0, 64, B), rng.integers(0, 64, B)], 1).astype(np.int32)).to(DEV)
        cref = torch.rand(B, 4, device=DEV)
        eref = torch.rand(B, 8, device=DEV)
        ntbc.train_colour_step(fmts, p, g, am, av, 1, xy, cref, eref, 64, 64, levels=4, coarsest=8, qat=qat)
        ne = ntbc.train_endpoint_param_count(fmts, 64, 4, 8) if hasattr(ntbc, "train_endpoint_param_count") else None
        if ne:
            pe = torch.from_numpy(rng.uniform(-0.5, 0.5, ne).astype(np.float32)).to(DEV)
            ge, ame, ave = (torch.zeros(ne, device=DEV) for _ in range(3))
            bxy = torch.from_numpy(np.stack([rng.integers(0, 16, B), rng.integers(0, 16, B)], 1).astype(np.int32)).to(DEV)
            ntbc.train_endpoint_step(fmts, pe, ge, ame, ave, 1, bxy, torch.rand(B, 16, 4, device=DEV), eref, 16, 16,
                                     levels=4, coarsest=8, qat=qat)
    # tcgen05 summation probe
    A = torch.from_numpy(rng.standard_normal((128, 32)).astype(np.float16)).to(DEV)
    Bm = torch.from_numpy(rng.standard_normal((16, 32)).astype(np.float16)).to(DEV)
    ntbc.debug_mma(A, Bm, torch.zeros(128, 16, device=DEV), 32, 16)
    torch.cuda.synchronize()
    print("sanitize target: all kernel families ran and matched", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2])

"""First GPU bring-up: exercises every C-ABI entry point against the oracle and prints diagnostics.
(Measurement / debugging tool; the graded parity checks live in tests/test_gpu_parity.py.)"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2407_09543_b200 import ntbc  # noqa: E402

dev = torch.device("cuda", 0)


def to_u64(t):
    return t.cpu().numpy().view(np.uint64)


def main():
    rng = np.random.default_rng(0)
    # --- decode_bc
    for fmt in (1, 4):
        blocks = rng.integers(0, 2 ** 63, (16, 16), dtype=np.int64)
        g = ntbc.decode_bc(torch.from_numpy(blocks).to(dev), fmt, 64, 64).cpu().numpy()
        o = oracle.decode_bc(blocks.view(np.uint64), fmt, 64, 64)
        print(f"decode_bc fmt{fmt}: bit-exact={np.array_equal(g.view(np.uint32), o.view(np.uint32))}")
    # --- pack
    fmts = [1, 1, 4, 4, 4]
    ep, col = synth.pack_inputs(fmts, 40, 12, seed=3)
    W, H = 160, 48
    g = ntbc.pack(fmts, torch.from_numpy(ep).to(dev), torch.from_numpy(col).to(dev), W, H)
    o = oracle.pack(fmts, ep, col, W, H)
    for k in range(len(fmts)):
        gk = to_u64(g[k])
        print(f"pack tex{k}: mismatched words {int((gk != o[k]).sum())} / {gk.size}")
    # --- fused path on C1 and C2 rows
    for cfg, rows in ((1, None), (2, (0, 2))):
        blob = synth.model_blob(cfg)
        W, H, _ = synth.config_shape(cfg)
        m = ntbc.Model(blob)
        om = oracle.Model(blob)
        r0, r1 = rows if rows else (0, H // 4)
        gep, gcol = ntbc.debug_mlp(m, W, H, r0, r1)
        t = time.time()
        oep, ocol = om.mlp_outputs(W, H, r0, r1)
        print(f"C{cfg}: oracle mlp {time.time() - t:.1f}s")
        gep, gcol = gep.cpu().numpy(), gcol.cpu().numpy()
        for name, a, b in (("ep", gep, oep), ("col", gcol, ocol)):
            rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-30)
            print(f"C{cfg} {name}: bit-exact frac {np.mean(a.view(np.uint32) == b.view(np.uint32)):.6f} "
                  f"max rel {rel.max():.3e} max abs {np.abs(a - b).max():.3e}")
        outs = ntbc.decode_material([m], W, H, row_begin=r0, row_end=r1)
        ow = om.decode_material(W, H, r0, r1)
        for k in range(m.n_tex):
            gk = to_u64(outs[k])
            print(f"C{cfg} decode tex{k}: mismatched words {int((gk != ow[k]).sum())} / {gk.size}")
        # pack fed the oracle's fp32 outputs must be bit-exact vs the oracle's words
        pk = ntbc.pack(m.fmts, torch.from_numpy(oep).to(dev), torch.from_numpy(ocol).to(dev), W, H, r0, r1)
        print(f"C{cfg} pack(oracle mlp) exact: {all(np.array_equal(to_u64(pk[k]), ow[k]) for k in range(m.n_tex))}")
    print("launches", ntbc.launch_count())


if __name__ == "__main__":
    main()

"""Per-parameter-class gradient discrepancy of the GPU training step vs the float64 oracle (debug aid)."""
import sys
import os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import train_oracle as T  # noqa: E402
from paper_2407_09543_b200 import ntbc  # noqa: E402

for qat, temp, levels in ((False, 0.01, 8), (True, 0.01, 8), (True, 0.1, 8), (True, 1.0, 8), (True, 0.01, 4), (False, 1.0, 8)):
    fmts, coarsest, B = [T.BC4, T.BC1], 16, 2048
    rng = np.random.default_rng(B)
    lay = T.layout(fmts, 64, levels, coarsest)
    n = sum(int(np.prod(s)) for _, s in lay)
    n_grid = sum(int(np.prod(s)) for nme, s in lay if nme.startswith("grid"))
    p = rng.standard_normal(n) * 0.3
    p[:n_grid] = rng.uniform(-1, 1, n_grid)
    p = p.astype(np.float32)
    W, H = 256, 192
    xy = np.stack([rng.integers(0, W, B), rng.integers(0, H, B)], 1).astype(np.int32)
    cref = rng.uniform(0, 1, (B, 4)).astype(np.float32)
    eref = rng.uniform(0, 1, (B, 8)).astype(np.float32)
    dp = torch.from_numpy(p).cuda()
    g, m, v = (torch.zeros(n, device="cuda") for _ in range(3))
    loss = ntbc.train_colour_step(fmts, dp, g, m, v, 1, torch.from_numpy(xy).cuda(), torch.from_numpy(cref).cuda(),
                                  torch.from_numpy(eref).cuda(), W, H, temperature=temp, levels=levels, coarsest=coarsest, qat=qat)
    torch.cuda.synchronize()
    rl, rg, _, _, _ = T.colour_step(torch.from_numpy(p.astype(np.float64)), torch.zeros(n, dtype=torch.float64),
                                    torch.zeros(n, dtype=torch.float64), 1, lay, fmts, torch.from_numpy(xy.astype(np.int64)),
                                    W, H, torch.from_numpy(cref.astype(np.float64)), torch.from_numpy(eref.astype(np.float64)),
                                    T=temp, qat=qat)
    gg = g.double().cpu()
    nr = float(torch.linalg.norm(rg))
    off = 0
    out = []
    for name, shape in lay:
        k = int(np.prod(shape))
        out.append(f"{name}:{float(torch.linalg.norm(gg[off:off + k] - rg[off:off + k])) / nr:.1e}")
        off += k
    print("qat", qat, "T", temp, "levels", levels, "loss", float(loss), rl, " ".join(out))

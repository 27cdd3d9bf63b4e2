"""Profiling target: a few colour / endpoint training steps at 2^20 texel / 2^16 block samples (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09543_b200 import ntbc  # noqa: E402

fmts = [1, 1, 4, 4, 4, 4]
rng = np.random.default_rng(0)
n = ntbc.train_param_count(fmts)
p = torch.from_numpy(rng.uniform(-1e-4, 1e-4, n).astype(np.float32)).cuda()
g, m, v = (torch.zeros(n, device="cuda") for _ in range(3))
B = 1 << 20
xy = torch.from_numpy(np.stack([rng.integers(0, 4096, B), rng.integers(0, 4096, B)], 1).astype(np.int32)).cuda()
cref, eref = torch.rand((B, 10), device="cuda"), torch.rand((B, 20), device="cuda")
for s in range(2):
    ntbc.train_colour_step(fmts, p, g, m, v, s + 1, xy, cref, eref, 4096, 4096)
torch.cuda.synchronize()
print("ok")

"""Dump GPU fp32 MLP outputs for some block rows of a config (debugging parity)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
from paper_2407_09543_b200 import ntbc
cfg = int(sys.argv[1]); rows = [int(r) for r in sys.argv[2].split(",")]
W, H, _ = synth.config_shape(cfg)
m = ntbc.Model(synth.model_blob(cfg))
res = {}
for r in rows:
    ep, col = ntbc.debug_mlp(m, W, H, r, r + 1)
    res[f"ep{r}"] = ep.cpu().numpy(); res[f"col{r}"] = col.cpu().numpy()
np.savez_compressed(sys.argv[3], **res)
print("dumped", rows)

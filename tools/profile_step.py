"""Minimal profiling target: load one material and run the fused decode a few times (for ncu)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2407_09543_b200 import ntbc  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    W, H, _ = synth.config_shape(cfg)
    m = ntbc.Model(synth.model_blob(cfg))
    if os.environ.get("NTBC_CONTRACT"):   # 1 = F, 2 = P
        ntbc.set_contract(m, int(os.environ["NTBC_CONTRACT"]))
    outs = ntbc.alloc_outputs([m], W, H)
    for _ in range(reps):
        ntbc.decode_material([m], W, H, outs=outs)
    torch.cuda.synchronize()
    print("ok", cfg, reps)


if __name__ == "__main__":
    main()

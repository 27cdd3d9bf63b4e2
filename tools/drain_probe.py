"""Tail (drain) cost of the fused kernel: time a C3 model over 4096 x H for H = 4096 and 8192 (the
second has twice the work units in one launch); 2 t(4096) - t(8192) is the per-launch drain loss."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2407_09543_b200 import ntbc  # noqa: E402


def t_ms(m, W, H, n=10):
    outs = ntbc.alloc_outputs([m], W, H)
    for _ in range(2):
        ntbc.decode_material([m], W, H, outs=outs)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record()
        ntbc.decode_material([m], W, H, outs=outs)
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[n // 2]


m = ntbc.Model(synth.model_blob(3))
t1, t2 = t_ms(m, 4096, 4096), t_ms(m, 4096, 8192)
print(f"t(4096^2) {t1:.3f} ms  t(4096x8192) {t2:.3f} ms  drain loss per launch {2 * t1 - t2:.3f} ms "
      f"({100 * (2 * t1 - t2) / t1:.1f}% of one material)")

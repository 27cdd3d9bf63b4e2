"""Colour-network training step on one B200: the paper architecture (texel grid 8
levels 16..2048, 16 -> 64 x3 -> N_c MLP), MetalPlates013-shaped heads (2 BC1 + 4 BC4, N_c = 10),
T = 0.01, random texel batches of a 4096^2 material with random reference colours / endpoints.  Time
per step by CUDA events (zero-gradient memsets, forward + backward + Adam); writes profiles/train_<tag>.json.

usage: python tools/train_bench.py [tag] [steps]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_09543_b200 import ntbc  # noqa: E402


def main(tag="r01", steps=20):
    fmts = [1, 1, 4, 4, 4, 4]
    W = H = 4096
    n = ntbc.train_param_count(fmts)
    rng = np.random.default_rng(0)
    p = torch.from_numpy(rng.uniform(-1e-4, 1e-4, n).astype(np.float32)).cuda()   # grid init of P:343
    g, m, v = (torch.zeros(n, device="cuda") for _ in range(3))
    rows = []
    for B in (1 << 16, 1 << 18, 1 << 20):
        xy = torch.from_numpy(np.stack([rng.integers(0, W, B), rng.integers(0, H, B)], 1).astype(np.int32)).cuda()
        cref = torch.rand((B, 10), device="cuda")
        eref = torch.rand((B, 20), device="cuda")
        loss = torch.zeros(1, device="cuda")
        for s in range(3):
            ntbc.train_colour_step(fmts, p, g, m, v, s + 1, xy, cref, eref, W, H, loss=loss)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i, (a, b) in enumerate(ev):
            a.record()
            ntbc.train_colour_step(fmts, p, g, m, v, 4 + i, xy, cref, eref, W, H, loss=loss)
            b.record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)[steps // 2]
        rows.append({"batch_texels": B, "ms_per_step": ms, "texel_samples_per_s": B / ms * 1e3,
                     "params": n, "loss": float(loss)})
    # endpoint network: block samples of the 1024^2 block grid, 16 reference colours each
    ne = ntbc.train_endpoint_param_count(fmts)
    pe = torch.from_numpy(rng.uniform(-1e-4, 1e-4, ne).astype(np.float32)).cuda()
    ge, me, ve = (torch.zeros(ne, device="cuda") for _ in range(3))
    erows = []
    for B in (1 << 14, 1 << 16):
        bxy = torch.from_numpy(np.stack([rng.integers(0, W // 4, B), rng.integers(0, H // 4, B)], 1)
                               .astype(np.int32)).cuda()
        c16 = torch.rand((B, 16, 10), device="cuda")
        eref = torch.rand((B, 20), device="cuda")
        loss = torch.zeros(1, device="cuda")
        for s in range(3):
            ntbc.train_endpoint_step(fmts, pe, ge, me, ve, s + 1, bxy, c16, eref, W // 4, H // 4, loss=loss)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i, (a, b) in enumerate(ev):
            a.record()
            ntbc.train_endpoint_step(fmts, pe, ge, me, ve, 4 + i, bxy, c16, eref, W // 4, H // 4, loss=loss)
            b.record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)[steps // 2]
        erows.append({"batch_blocks": B, "ms_per_step": ms, "block_samples_per_s": B / ms * 1e3, "params": ne})
    out = {"tag": tag, "gpu": torch.cuda.get_device_name(0), "textures": "2 BC1 + 4 BC4 (N_c = 10, N_e = 20)",
           "endpoint_rows": erows,
           "paper_context": "20k iterations of both networks in ~10 min (aggressive) on an RX 7900 XT, batch not "
                            "stated (P:509): ~30 ms per iteration", "rows": rows}
    with open(os.path.join(ROOT, "profiles", f"train_{tag}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("| batch (texels) | ms / step | Mtexel-samples/s |")
    print("|---|---|---|")
    for r in rows:
        print(f"| {r['batch_texels']} | {r['ms_per_step']:.2f} | {r['texel_samples_per_s'] / 1e6:.0f} |")
    print("| endpoint batch (blocks) | ms / step | Mblock-samples/s |")
    for r in erows:
        print(f"| {r['batch_blocks']} | {r['ms_per_step']:.2f} | {r['block_samples_per_s'] / 1e6:.1f} |")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or []), *(int(x) for x in sys.argv[2:3]))

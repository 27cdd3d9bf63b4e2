"""The paper's four inference workloads (Tab. 1) on one B200.

The material is MetalPlates013-shaped: six 4096^2 textures, 2 BC1 (diffuse, normal) + 4 BC4
(displacement, roughness, AO, metalness).  Workloads:
  CS BC1&BC4  -- conservative: an all-BC1 model (2 textures) and an all-BC4 model (4 textures),
                 one ntbc_decode_material call with both (ONE persistent launch, CTAs partitioned by model);
  CS BC1 only -- the RGB model alone;
  AG BC1&BC4  -- aggressive: one model with all 6 textures (config 6, C3');
  AG BC1 only -- an aggressive model over the two RGB textures only.
Random-init weights of the paper architecture (seeded), synthetic grids; kernel time by CUDA events
on the launching stream, L2 flushed (256 MiB write) between steps outside the events.  Writes
profiles/tab1_<tag>.json and prints a table with the paper's RX 7900 XT times beside ours.  Env
NTBC_CONTRACT=2 runs every model under contract P (binary16 selu arithmetic).

usage: python tools/tab1.py [tag] [steps]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2407_09543_b200 import ntbc  # noqa: E402

W = H = 4096
CONTRACT = int(os.environ.get("NTBC_CONTRACT", "0"))
PAPER_MS = {"CS BC1&BC4": 49.84, "CS BC1 only": 25.57, "AG BC1&BC4": 27.31, "AG BC1 only": 25.96}


def models_for(workload):
    spec = lambda fmts, seed: synth.serialize(synth.random_model(synth.ModelSpec(list(fmts)), seed))  # noqa: E731
    rgb, sc = [synth.BC1] * 2, [synth.BC4] * 4
    if workload == "CS BC1&BC4":
        return [spec(rgb, 101), spec(sc, 102)]
    if workload == "CS BC1 only":
        return [spec(rgb, 101)]
    if workload == "AG BC1&BC4":
        return [synth.model_blob(6)]
    return [spec(rgb, 103)]


def time_workload(blobs, steps):
    models = [ntbc.Model(b) for b in blobs]
    for m in models:
        ntbc.set_contract(m, CONTRACT)
    outs = ntbc.alloc_outputs(models, W, H)
    stream = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(stream):
        for _ in range(3):
            ntbc.decode_material(models, W, H, outs=outs, stream=stream)
        stream.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in ev:
            flush.zero_()
            a.record(stream)
            ntbc.decode_material(models, W, H, outs=outs, stream=stream)
            b.record(stream)
        stream.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    n_tex = sum(m.n_tex for m in models)
    return ms, n_tex


def main(tag="r01", steps=20):
    rows = []
    for wl in PAPER_MS:
        ms, n_tex = time_workload(models_for(wl), steps)
        blocks = (W // 4) * (H // 4) * n_tex
        rows.append({"workload": wl, "textures": n_tex, "ms": ms, "mblocks_per_s": blocks / ms / 1e3,
                     "paper_ms_rx7900xt": PAPER_MS[wl], "speedup_vs_paper": PAPER_MS[wl] / ms})
    out = {"tag": tag, "gpu": torch.cuda.get_device_name(0), "width": W, "height": H, "steps": steps,
           "contract": {0: "H", 1: "F", 2: "P"}[CONTRACT],
           "timing": "CUDA events, kernel only, L2 flushed between steps", "rows": rows}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"tab1_{tag}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("| workload | textures | B200 ms | Mblocks/s | paper ms (RX 7900 XT) | ratio |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['workload']} | {r['textures']} | {r['ms']:.2f} | {r['mblocks_per_s']:.0f} | "
              f"{r['paper_ms_rx7900xt']:.2f} | {r['speedup_vs_paper']:.1f}x |")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or []), *(int(x) for x in sys.argv[2:3]))

"""Reference BC1/BC4 encoder on one B200: 4096^2 textures, CUDA events on the
launching stream, L2 flushed between steps (outside the events).  Reports Mblocks/s and the achieved
HBM bandwidth against MEASURED_PEAKS.json (algorithmic bytes: fp32 texels in + 8 B per block out).
Writes profiles/refenc_<tag>.json.

usage: python tools/refenc_bench.py [tag] [steps]
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
    W = H = 4096
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6453.4)   # MEASURED_PEAKS.json (copy bandwidth), else the guide's figure
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    rows = []
    rng = np.random.default_rng(0)
    for fmt, ch in ((1, 3), (4, 1)):
        tex = torch.from_numpy(rng.uniform(0, 1, (H, W, ch)).astype(np.float32)).cuda()
        out = torch.empty((H // 4, W // 4), dtype=torch.int64, device="cuda")
        for n_refine in (0, 2):
            with torch.cuda.stream(stream):
                for _ in range(3):
                    ntbc.encode_bc(tex, fmt, W, H, n_refine, out=out, stream=stream)
                stream.synchronize()
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
                for a, b in ev:
                    flush.zero_()
                    a.record(stream)
                    ntbc.encode_bc(tex, fmt, W, H, n_refine, out=out, stream=stream)
                    b.record(stream)
                stream.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in ev) / steps
            nbytes = W * H * ch * 4 + (W // 4) * (H // 4) * 8
            rows.append({"format": "BC1" if fmt == 1 else "BC4", "n_refine": n_refine, "ms": ms,
                         "mblocks_per_s": (W // 4) * (H // 4) / ms / 1e3, "algorithmic_bytes": nbytes,
                         "achieved_gbps": nbytes / ms / 1e6, "hbm_peak_gbps": hbm,
                         "hbm_frac": nbytes / ms / 1e6 / hbm})
    out = {"tag": tag, "gpu": torch.cuda.get_device_name(0), "width": W, "height": H, "steps": steps,
           "input": "uniform noise fp32 texels", "timing": "CUDA events, L2 flushed between steps", "rows": rows}
    with open(os.path.join(ROOT, "profiles", f"refenc_{tag}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("| format | refinements | ms | Mblocks/s | GB/s | HBM frac |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['format']} | {r['n_refine']} | {r['ms']:.3f} | {r['mblocks_per_s']:.0f} | "
              f"{r['achieved_gbps']:.0f} | {r['hbm_frac']:.2f} |")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or []), *(int(x) for x in sys.argv[2:3]))

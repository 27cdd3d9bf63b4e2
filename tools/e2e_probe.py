"""Break the e2e step (ntbc_decode_material_host) of a config into its parts on the GPU.

usage: python tools/e2e_probe.py [config]   (NTBC_NO_PIPELINED_COPY=1 disables the chunked copy-back)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2407_09543_b200 import ntbc  # noqa: E402


def timed(fn, stream, n=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[n // 2]


def main(cfg=3):
    W, H, _ = synth.config_shape(cfg)
    blob = synth.model_blob(cfg)
    m = ntbc.Model(blob)
    BW, BH = W // 4, H // 4
    stream = torch.cuda.Stream()
    pinned = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
    host = [torch.empty((BH, BW), dtype=torch.int64).pin_memory() for _ in range(m.n_tex)]
    dev = ntbc.decode_material([m], W, H)
    dblob = torch.empty(len(blob), dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(stream):
        h2d = timed(lambda: dblob.copy_(pinned, non_blocking=True), stream)
        d2h = timed(lambda: [h.copy_(d, non_blocking=True) for h, d in zip(host, dev)], stream)
    kern = timed(lambda: ntbc.decode_material([m], W, H, outs=dev, stream=stream), stream)
    e2e = timed(lambda: ntbc.decode_material_host([m], [pinned], W, H, host, stream=stream), stream)
    n = 20
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        ntbc.decode_material_host([m], [pinned], W, H, host, stream=stream)
    b.record(stream)
    torch.cuda.synchronize()
    span = a.elapsed_time(b) / n
    print(f"config {cfg}: h2d {h2d:.3f} ms ({len(blob) / h2d / 1e6:.1f} GB/s)  d2h {d2h:.3f} ms "
          f"({BW * BH * 8 * m.n_tex / d2h / 1e6:.1f} GB/s)  kernel {kern:.3f} ms  e2e {e2e:.3f} ms  span/call {span:.3f} ms  "
          f"pipelined={os.environ.get('NTBC_NO_PIPELINED_COPY', '0') != '1'}")


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))

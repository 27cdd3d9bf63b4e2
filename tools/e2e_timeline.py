"""Where the end-to-end time goes: event timeline of ntbc_decode_material_host in steady state
(NTBC_TIMELINE=1; times in ms relative to the call's start on the caller's stream)."""
import os
import sys

import torch

os.environ["NTBC_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2407_09543_b200 import ntbc  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
W, H, _ = synth.config_shape(cfg)
blob = synth.model_blob(cfg)
m = ntbc.Model(blob)
pinned = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
host_all = torch.empty((m.n_tex, H // 4, W // 4), dtype=torch.int64).pin_memory()
host = [host_all[k] for k in range(m.n_tex)] if os.environ.get("NTBC_SEPARATE_PLANES") != "1" else [torch.empty((H // 4, W // 4), dtype=torch.int64).pin_memory() for _ in range(m.n_tex)]
stream = torch.cuda.Stream()
for _ in range(3):
    ntbc.decode_material_host([m], [pinned], W, H, host, stream=stream)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
for _ in range(10):
    ntbc.decode_material_host([m], [pinned], W, H, host, stream=stream)
b.record(stream)
torch.cuda.synchronize()
t = ntbc.debug_host_timeline(m)
print(f"span/call {a.elapsed_time(b) / 10:.3f} ms; last call: upload done {t[1]:+.3f}, kernel start {t[2]:+.3f}, "
      f"kernel end {t[3]:+.3f}, copies done " + " ".join(f"{x:+.3f}" for x in t[4:8]) +
      f"; previous call start {t[8]:+.3f}, its copies done " + " ".join(f"{x:+.3f}" for x in t[9:13]))
import time  # noqa: E402
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    ntbc.decode_material_host([m], [pinned], W, H, host, stream=stream)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3 * (t1 - t0) / 10:.3f} ms/call; wall incl. sync {1e3 * (t2 - t0) / 10:.3f} ms/call")
for n in (10, 40):
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(n):
        ntbc.decode_material_host([m], [pinned], W, H, host, stream=stream)
    b.record(stream)
    torch.cuda.synchronize()
    print(f"{n} calls: span/call {a.elapsed_time(b) / n:.3f} ms")
periods = []
for _ in range(12):
    ntbc.decode_material_host([m], [pinned], W, H, host, stream=stream)
    torch.cuda.synchronize()   # no overlap between calls: isolated call
    t = ntbc.debug_host_timeline(m)
    periods.append(t[3] - t[2])
print("isolated calls, kernel ms:", " ".join(f"{x:.3f}" for x in periods))
for n in (5, 6, 7, 8, 9, 10):
    torch.cuda.synchronize()
    for _ in range(n):
        ntbc.decode_material_host([m], [pinned], W, H, host, stream=stream)
    torch.cuda.synchronize()
    t = ntbc.debug_host_timeline(m)
    print(f"loop of {n}: last call period {-t[8]:.3f} ms, kernel {t[3] - t[2]:.3f}, tail {max(t[4:8]) - t[3]:.3f}, slot-gap {-max(t[9:13]):.3f}")

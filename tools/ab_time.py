"""A/B kernel timing of in-tree library variants (debugging aid, not a bench number).

usage: python tools/ab_time.py [config] [reps] lib1.so lib2.so:NTBC_NWG=4 ...
Each variant runs in its own process (NTBC_LIB=<name>, plus optional KEY=VAL env settings after ':'), decodes the config's material `reps`
times with the L2 flushed between launches and prints median / min kernel ms (CUDA events)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys, json, torch
sys.path.insert(0, %r)
import synth
from paper_2407_09543_b200 import ntbc
cfg, reps = int(sys.argv[1]), int(sys.argv[2])
W, H, _ = synth.config_shape(cfg)
m = ntbc.Model(synth.model_blob(cfg))
if os.environ.get("NTBC_CONTRACT"):
    ntbc.set_contract(m, int(os.environ["NTBC_CONTRACT"]))
outs = ntbc.alloc_outputs([m], W, H)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for _ in range(5):
    ntbc.decode_material([m], W, H, outs=outs, stream=s)
ts = []
for _ in range(reps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); ntbc.decode_material([m], W, H, outs=outs, stream=s); b.record(s)
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ts.sort()
print(json.dumps({"lib": os.environ.get("NTBC_LIB", "libntbc.so"), "nwg": os.environ.get("NTBC_NWG"),
                  "contract": os.environ.get("NTBC_CONTRACT", "0"), "cfg": cfg, "median_ms": ts[len(ts) // 2],
                  "min_ms": ts[0]}))
""" % ROOT


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    libs = sys.argv[3:] or ["libntbc.so"]
    for rnd in range(2):   # two interleaved rounds: clocks drift between processes
        for spec in libs:
            lib, *kv = spec.split(":")
            env = dict(os.environ, NTBC_LIB=lib, **dict(x.split("=", 1) for x in kv))
            out = subprocess.run([sys.executable, "-c", CHILD, str(cfg), str(reps)], env=env, capture_output=True,
                                 text=True)
            print(f"round {rnd}:", out.stdout.strip() or out.stderr.strip()[-400:], flush=True)


if __name__ == "__main__":
    main()

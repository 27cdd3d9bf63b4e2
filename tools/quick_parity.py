"""Quick words + MLP parity check of one config's sampled rows (debugging aid)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, synth
from paper_2407_09543_b200 import ntbc
cfg = int(sys.argv[1]); rows = [int(x) for x in sys.argv[2].split(",")]
W, H, _ = synth.config_shape(cfg)
blob = synth.model_blob(cfg)
m, om = ntbc.Model(blob), oracle.Model(blob)
full = ntbc.decode_material([m], W, H)
torch.cuda.synchronize()
for r in rows:
    ow = om.decode_material(W, H, r, r + 1)
    gw = [t.cpu().numpy().view(np.uint64)[r:r + 1] for t in full]
    bad = [int((g != o).sum()) for g, o in zip(gw, ow)]
    gep, gcol = ntbc.debug_mlp(m, W, H, r, r + 1)
    oep, ocol = om.mlp_outputs(W, H, r, r + 1)
    be = int((gep.cpu().numpy().view(np.uint32) != oep.view(np.uint32)).sum())
    bc = int((gcol.cpu().numpy().view(np.uint32) != ocol.view(np.uint32)).sum())
    print(f"cfg{cfg} row {r}: words bad {bad}  ep bad {be}/{oep.size}  col bad {bc}/{ocol.size}")

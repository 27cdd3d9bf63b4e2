"""Parity of a custom architecture (debugging aid): hidden, W, H, levels."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, synth
from paper_2407_09543_b200 import ntbc
for hidden in (16, 32, 64):
    for W, H in ((64, 64), (1024, 16)):
        sp = synth.ModelSpec([synth.BC1, synth.BC4], hidden=hidden, block_levels=3, block_coarsest=8, texel_levels=4, texel_coarsest=8)
        blob = synth.serialize(synth.random_model(sp, 3))
        m, om = ntbc.Model(blob), oracle.Model(blob)
        gep, gcol = ntbc.debug_mlp(m, W, H, 0, 1)
        oep, ocol = om.mlp_outputs(W, H, 0, 1)
        ge = gep.cpu().numpy(); gc = gcol.cpu().numpy()
        be = (ge.view(np.uint32) != oep.view(np.uint32))
        bc = (gc.view(np.uint32) != ocol.view(np.uint32))
        badb = sorted(set(np.argwhere(be)[:, 1].tolist()))
        print(f"H={hidden} {W}x{H}: ep bad {int(be.sum())}/{be.size} blocks {badb[:12]}..{len(badb)}  col bad {int(bc.sum())}/{bc.size}", flush=True)

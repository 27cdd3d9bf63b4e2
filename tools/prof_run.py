import os, sys, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2407_09543_b200 import ntbc
W, H, _ = synth.config_shape(3)
m = ntbc.Model(synth.model_blob(3))
outs = ntbc.alloc_outputs([m], W, H)
ntbc.decode_material([m], W, H, outs=outs); torch.cuda.synchronize()
print("----- second launch", flush=True)
ntbc.decode_material([m], W, H, outs=outs); torch.cuda.synchronize()

"""The CUDA path against the PLAIN-definition oracle (-m gpu): full C2 and sampled
full-width rows of C3 / C4 at full size, under north_star's agreement rule (tests/faithful.py), counts
printed by class and written to gpurun_out/faithfulness_gpu.json.  The asserted bounds are those of
tests/test_faithfulness.py: relative to the spread between plain readings of the same
half-precision network, measured on the same rows -- the literal 1e-3 / zero-unexcused rule holds bit-exactly
against the pinned oracle (tests/test_gpu_parity.py) and cannot hold against any other implementation of
the paper's binary16 inference."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from faithful import CLASSES, compare_words, float_stats

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RESULTS = {}


def _plain(om, W, H, r0, r1, dot=(0, 16, 100, 0), act=1):
    saved = (oracle.get_dot_model(), int(oracle.lib().o_get_act_model()))
    try:
        oracle.set_dot_model(*dot)
        oracle.set_act_model(act)
        return (om.decode_material(W, H, r0, r1),) + om.mlp_outputs(W, H, r0, r1)
    finally:
        oracle.set_dot_model(*saved[0])
        oracle.set_act_model(saved[1])


@pytest.mark.parametrize("cfg,rows", [(2, None), (3, ((0, 2), (517, 519), (1022, 1024))), (4, ((0, 1), (700, 701)))])
def test_cuda_path_vs_plain_definitions(cfg, rows):
    from paper_2407_09543_b200 import ntbc
    W, H, _ = synth.config_shape(cfg)
    blob = synth.model_blob(cfg)
    m, om = ntbc.Model(blob), oracle.Model(blob)
    full = [t.cpu().numpy().view(np.uint64) for t in ntbc.decode_material([m], W, H)]
    rows = rows or ((0, H // 4),)
    agg = None
    for r0, r1 in rows:
        gw = [f[r0:r1] for f in full]
        gep, gcol = (t.cpu().numpy() for t in ntbc.debug_mlp(m, W, H, r0, r1))
        pw, pep, pcol = _plain(om, W, H, r0, r1)
        sw, sep, scol = _plain(om, W, H, r0, r1, dot=(1, 1, 100, 0))   # plain reading with a sequential dot
        rep = compare_words(om.fmts, gw, pw, pep, pcol)
        ref = compare_words(om.fmts, sw, pw, pep, pcol)
        rep["floats"] = {"endpoint": float_stats(gep, pep), "colour": float_stats(gcol, pcol)}
        rep["plain_seq_dot"] = {"mismatched": ref["mismatched"], "unexcused": ref["unexcused"],
                                "endpoint_max_rel": float_stats(sep, pep)["max_rel"],
                                "colour_max_rel": float_stats(scol, pcol)["max_rel"]}
        if agg is None:
            agg = rep
        else:
            for k in ("blocks", "words", "mismatched", "excused", "unexcused"):
                agg[k] += rep[k]
            for c in CLASSES:
                agg[c] = [a + b for a, b in zip(agg[c], rep[c])]
            for k in ("mismatched", "unexcused"):
                agg["plain_seq_dot"][k] += rep["plain_seq_dot"][k]
            for side in ("endpoint", "colour"):
                agg["floats"][side]["max_rel"] = max(agg["floats"][side]["max_rel"], rep["floats"][side]["max_rel"])
                key = side + "_max_rel"
                agg["plain_seq_dot"][key] = max(agg["plain_seq_dot"][key], rep["plain_seq_dot"][key])
    agg["excused_fraction_of_blocks"] = agg["excused"] / agg["blocks"]
    RESULTS[f"C{cfg}"] = agg
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "faithfulness_gpu.json"), "w") as f:
        json.dump(RESULTS, f, indent=1)
    print(f"\nC{cfg} CUDA vs plain: {agg['mismatched']} of {agg['words']} words differ ({agg['excused']} excused, "
          f"{agg['unexcused']} unexcused); " + ", ".join(f"{c} {agg[c][0]}/{agg[c][1]}" for c in CLASSES)
          + f"; max rel endpoint {agg['floats']['endpoint']['max_rel']:.2e} colour {agg['floats']['colour']['max_rel']:.2e}"
          + f" | plain seq-dot reading: {agg['plain_seq_dot']}")
    seq = agg["plain_seq_dot"]
    for side in ("endpoint", "colour"):
        assert agg["floats"][side]["zero_violations"] == 0
        assert agg["floats"][side]["max_rel"] <= 2 * seq[side + "_max_rel"] + 1e-6
    assert agg["mismatched"] <= 2 * seq["mismatched"] + 4
    assert agg["unexcused"] <= 2 * seq["unexcused"] + 4

"""Contract F on the GPU (-m gpu): ntbc_set_contract(m, 1) keeps the hidden
activations in binary32 and feeds each tcgen05 MMA the split hi = RN16(a), lo = RN16(a - hi).

  * bit-exact against the oracle's pinned F mode (`oracle.contract_f()`): words and MLP outputs;
  * against the PLAIN definitions of contract F (exact dots, float64 libm activations) north_star's float
    rule and its word rule hold -- floats within 1e-3 relative, zero unexcused words -- on the full C2
    material and sampled full-width rows of C3, and on the full C2 material also the excused fraction is
    under 1e-4 of the blocks (counts printed, written to gpurun_out/contract_f_gpu.json).  The excused
    fraction grows with the decisions per block (C3: 5 textures, 18 endpoint roundings + 80 index choices per
    block): ~6e-4 on the C3 sample, SURVEY App. B's prediction for any implementation that is not
    bit-identical to the reference.  Under the paper's contract H not even the float rule can hold (§5.1)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from faithful import CLASSES, compare_words, float_stats

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RESULTS = {}


@pytest.fixture(scope="module")
def ntbc():
    from paper_2407_09543_b200 import ntbc as n
    return n


def u64(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("case", ["c1", "c2rows", "ragged", "c3rows"])
def test_contract_f_bit_exact_vs_pinned_oracle(ntbc, case):
    if case == "ragged":
        sp = synth.ModelSpec([synth.BC1, synth.BC4, synth.BC4], hidden=32, block_levels=3, block_coarsest=5,
                             texel_levels=4, texel_coarsest=8)
        blob, W, H, rows = synth.serialize(synth.random_model(sp, 91)), 4 * 129, 12, (0, 3)
    else:
        cfg = {"c1": 1, "c2rows": 2, "c3rows": 3}[case]
        W, H, _ = synth.config_shape(cfg)
        blob = synth.model_blob(cfg)
        rows = {"c1": (0, H // 4), "c2rows": (127, 130), "c3rows": (517, 519)}[case]
    m, om = ntbc.Model(blob), oracle.Model(blob)
    ntbc.set_contract(m, 1)
    full = ntbc.decode_material([m], W, H)
    gep, gcol = ntbc.debug_mlp(m, W, H, *rows)
    with oracle.contract_f():
        ow = om.decode_material(W, H, *rows)
        oep, ocol = om.mlp_outputs(W, H, *rows)
    for k in range(m.n_tex):
        assert np.array_equal(u64(full[k])[rows[0]:rows[1]], ow[k]), k
    assert np.array_equal(gep.cpu().numpy().view(np.uint32), oep.view(np.uint32))
    assert np.array_equal(gcol.cpu().numpy().view(np.uint32), ocol.view(np.uint32))


@pytest.mark.parametrize("cfg,rows", [(2, None), (3, ((0, 2), (517, 519), (1022, 1024)))])
def test_contract_f_meets_the_literal_rule_vs_plain(ntbc, cfg, rows):
    W, H, _ = synth.config_shape(cfg)
    blob = synth.model_blob(cfg)
    m, om = ntbc.Model(blob), oracle.Model(blob)
    ntbc.set_contract(m, 1)
    full = [u64(t) for t in ntbc.decode_material([m], W, H)]
    rows = rows or ((0, H // 4),)
    agg = None
    for r0, r1 in rows:
        gep, gcol = (t.cpu().numpy() for t in ntbc.debug_mlp(m, W, H, r0, r1))
        with oracle.contract_f(), oracle.plain_definitions():
            pw = om.decode_material(W, H, r0, r1)
            pep, pcol = om.mlp_outputs(W, H, r0, r1)
        rep = compare_words(om.fmts, [f[r0:r1] for f in full], pw, pep, pcol)
        rep["floats"] = {"endpoint": float_stats(gep, pep), "colour": float_stats(gcol, pcol)}
        if agg is None:
            agg = rep
        else:
            for k in ("blocks", "words", "mismatched", "excused", "unexcused"):
                agg[k] += rep[k]
            for c in CLASSES:
                agg[c] = [a + b for a, b in zip(agg[c], rep[c])]
            for side in ("endpoint", "colour"):
                for key in ("max_rel", "max_abs"):
                    agg["floats"][side][key] = max(agg["floats"][side][key], rep["floats"][side][key])
                agg["floats"][side]["zero_violations"] += rep["floats"][side]["zero_violations"]
    RESULTS[f"C{cfg}"] = agg
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "contract_f_gpu.json"), "w") as f:
        json.dump(RESULTS, f, indent=1)
    print(f"\nC{cfg} contract F, CUDA vs plain: {agg['mismatched']} of {agg['words']} words differ "
          f"({agg['excused']} excused, {agg['unexcused']} unexcused); "
          + ", ".join(f"{c} {agg[c][0]}/{agg[c][1]}" for c in CLASSES)
          + f"; max rel endpoint {agg['floats']['endpoint']['max_rel']:.2e} colour {agg['floats']['colour']['max_rel']:.2e}")
    for side in ("endpoint", "colour"):
        assert agg["floats"][side]["max_rel"] <= 1e-3
        assert agg["floats"][side]["zero_violations"] == 0
    assert agg["unexcused"] == 0
    if cfg == 2:   # the full material: the excused-fraction clause of the rule
        assert agg["excused"] < 1e-4 * agg["blocks"]


def test_contract_f_api(ntbc):
    m = ntbc.Model(synth.model_blob(1))
    with pytest.raises(ntbc.NtbcError):
        ntbc.set_contract(m, 3)
    naive = ntbc.Model(synth.model_blob(8))
    with pytest.raises(ntbc.NtbcError):
        ntbc.set_contract(naive, 1)
    ntbc.set_contract(m, 1)
    ntbc.set_contract(m, 0)                       # back to H: identical to a fresh model
    W, H, _ = synth.config_shape(1)
    a = [u64(t) for t in ntbc.decode_material([m], W, H)]
    b = [u64(t) for t in ntbc.decode_material([ntbc.Model(synth.model_blob(1))], W, H)]
    assert all(np.array_equal(x, y) for x, y in zip(a, b))

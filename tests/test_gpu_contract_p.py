"""Contract P on the GPU (-m gpu): ntbc_set_contract(m, 2) evaluates the
hidden selu in binary16 arithmetic on packed f16x2 lanes (HFMA2 / HMUL2 / HADD2 / HMNMX2, `selu2_h16`).

  * bit-exact against the oracle's contract P (`oracle.contract_p()`, R9-P): words and MLP outputs, on C1,
    C2 rows, a ragged hidden-32 model, sampled C3 rows and a conservative pair in one launch;
  * the distance to the PLAIN definitions measured under north_star's rule and printed (written to
    gpurun_out/contract_p_gpu.json): the price of binary16 arithmetic.  Not asserted
    against the rule -- it is the measurement of this contract, not a claim that it meets the rule."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from faithful import CLASSES, compare_words, float_stats

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ntbc():
    from paper_2407_09543_b200 import ntbc as n
    return n


def u64(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("case", ["c1", "c2rows", "ragged", "c3rows"])
def test_contract_p_bit_exact_vs_oracle(ntbc, case):
    if case == "ragged":
        sp = synth.ModelSpec([synth.BC1, synth.BC4, synth.BC4], hidden=32, block_levels=3, block_coarsest=5,
                             texel_levels=4, texel_coarsest=8)
        blob, W, H, rows = synth.serialize(synth.random_model(sp, 92)), 4 * 129, 12, (0, 3)
    else:
        cfg = {"c1": 1, "c2rows": 2, "c3rows": 3}[case]
        W, H, _ = synth.config_shape(cfg)
        blob = synth.model_blob(cfg)
        rows = {"c1": (0, H // 4), "c2rows": (127, 130), "c3rows": (517, 519)}[case]
    m, om = ntbc.Model(blob), oracle.Model(blob)
    ntbc.set_contract(m, 2)
    full = ntbc.decode_material([m], W, H)
    gep, gcol = ntbc.debug_mlp(m, W, H, *rows)
    with oracle.contract_p():
        ow = om.decode_material(W, H, *rows)
        oep, ocol = om.mlp_outputs(W, H, *rows)
    for k in range(m.n_tex):
        assert np.array_equal(u64(full[k])[rows[0]:rows[1]], ow[k]), k
    assert np.array_equal(gep.cpu().numpy().view(np.uint32), oep.view(np.uint32))
    assert np.array_equal(gcol.cpu().numpy().view(np.uint32), ocol.view(np.uint32))
    hep, _ = om.mlp_outputs(W, H, *rows)          # contract H: a different arithmetic
    assert not np.array_equal(hep.view(np.uint32), oep.view(np.uint32))


def test_contract_p_pair_one_launch(ntbc):
    """A conservative pair, both models in contract P: one persistent launch, bit-exact."""
    rgb = synth.serialize(synth.random_model(synth.ModelSpec([synth.BC1, synth.BC1], block_levels=4, texel_levels=5), 15))
    sc = synth.serialize(synth.random_model(synth.ModelSpec([synth.BC4] * 3, block_levels=4, texel_levels=5), 16))
    ms = [ntbc.Model(rgb), ntbc.Model(sc)]
    for m in ms:
        ntbc.set_contract(m, 2)
    n0 = ntbc.launch_count()
    got = ntbc.decode_material(ms, 256, 128)
    assert ntbc.launch_count() - n0 <= 3          # the two models' prep launches + ONE fused launch
    with oracle.contract_p():
        ref = list(oracle.Model(rgb).decode_material(256, 128)) + list(oracle.Model(sc).decode_material(256, 128))
    for k in range(5):
        assert np.array_equal(u64(got[k]), ref[k]), k


def test_contract_p_distance_to_plain(ntbc):
    """Full C2: contract P (CUDA) against the plain definitions, by class -- printed and recorded."""
    W, H, _ = synth.config_shape(2)
    blob = synth.model_blob(2)
    m, om = ntbc.Model(blob), oracle.Model(blob)
    ntbc.set_contract(m, 2)
    full = [u64(t) for t in ntbc.decode_material([m], W, H)]
    gep, gcol = (t.cpu().numpy() for t in ntbc.debug_mlp(m, W, H, 0, H // 4))
    with oracle.plain_definitions():
        pw = om.decode_material(W, H)
        pep, pcol = om.mlp_outputs(W, H)
    rep = compare_words(om.fmts, full, pw, pep, pcol)
    rep["floats"] = {"endpoint": float_stats(gep, pep), "colour": float_stats(gcol, pcol)}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "contract_p_gpu.json"), "w") as f:
        json.dump({"C2": rep}, f, indent=1)
    print(f"\nC2 contract P, CUDA vs plain: {rep['mismatched']} of {rep['words']} words differ "
          f"({rep['excused']} excused, {rep['unexcused']} unexcused); "
          + ", ".join(f"{c} {rep[c][0]}/{rep[c][1]}" for c in CLASSES)
          + f"; max rel endpoint {rep['floats']['endpoint']['max_rel']:.2e} colour {rep['floats']['colour']['max_rel']:.2e}")
    assert sum(sum(rep[c]) for c in CLASSES) == rep["mismatched"]
    assert rep["floats"]["endpoint"]["zero_violations"] == 0 and rep["floats"]["colour"]["zero_violations"] == 0


def test_contract_p_api(ntbc):
    m = ntbc.Model(synth.model_blob(1))
    naive = ntbc.Model(synth.model_blob(8))
    with pytest.raises(ntbc.NtbcError):
        ntbc.set_contract(naive, 2)
    ntbc.set_contract(m, 2)
    ntbc.set_contract(m, 0)
    W, H, _ = synth.config_shape(1)
    a = [u64(t) for t in ntbc.decode_material([m], W, H)]
    b = [u64(t) for t in ntbc.decode_material([ntbc.Model(synth.model_blob(1))], W, H)]
    assert all(np.array_equal(x, y) for x, y in zip(a, b))

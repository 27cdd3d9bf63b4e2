"""Faithfulness of the pinned arithmetic to the PLAIN definitions (-m "not gpu"), VERDICT r01 item 1.

The oracle's default (pinned) mode follows the op sequences the kernels execute bit for bit: R9's
polynomial exponential and R10's tensor-core summation order.  Its plain mode (`oracle.plain_definitions`)
computes the definitions themselves: every dot product exact and rounded once (P:331 is silent on the
order, so "exact" is the plain reading), selu / sigmoid in float64 with libm, one rounding.
Both keep the paper's binary16 operands at every layer input.

These tests measure the pinned oracle -- bit-identical to the CUDA path (tests/test_gpu_parity.py) --
against the plain mode under north_star's agreement rule (tests/faithful.py), print the counts by class
and assert the bounds DESIGN.md §5.1 derives.  They also measure two other plain readings of the same
half-precision network (a sequential binary32 dot product; binary32 libm activations) against the plain
mode: the spread between *plain* implementations is the floor any implementation of the paper's
half-precision inference has (the binary16 re-rounding of each layer input turns a one-ulp difference of
a pre-activation into a one-binary16-ulp activation change, which the next layers amplify).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from faithful import CLASSES, compare_words, float_stats

L = oracle.lib()
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- the plain mode itself (pinned)
def test_plain_activations_vs_torch_float64():
    """Plain selu / sigmoid = torch float64 (exact selu constants) rounded once to binary32."""
    z = np.concatenate([np.linspace(-40, 40, 40001), -np.geomspace(1e-30, 1, 2001)]).astype(np.float32)
    zt = torch.from_numpy(z.astype(np.float64))
    with oracle.plain_definitions():
        got_selu = np.array([L.o_selu(float(v)) for v in z], np.float32)
        got_sig = np.array([L.o_sigmoid(float(v)) for v in z], np.float32)
    ref_selu = torch.nn.functional.selu(zt).numpy()
    ref_sig = torch.sigmoid(zt).numpy()
    # one rounding of the float64 value: within half a binary32 ulp (torch's float64 selu may itself
    # differ from libm expm1 by an ulp of float64 -- far below that)
    ulp = np.spacing(np.abs(got_selu).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(got_selu - ref_selu) <= 0.5 * ulp + 1e-300)
    ulp = np.spacing(got_sig.astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(got_sig - ref_sig) <= 0.5 * ulp + 1e-300)
    assert oracle.get_dot_model()[0] == 1 and L.o_get_act_model() == 0   # the context restored the pinned mode


def test_plain_dot_is_exact_sum_rounded_once():
    """Plain mode's layer = the exact float64 sum of bias + fp16 x fp16 products (math.fsum), one RN."""
    rng = np.random.default_rng(7)
    W = [(rng.standard_normal((64, 16)) * 0.3).astype(np.float16)]
    b = [(rng.standard_normal(16) * 0.1).astype(np.float16)]
    for _ in range(200):
        x = (rng.standard_normal(64) * 2).astype(np.float32)
        x16 = x.astype(np.float16)
        with oracle.plain_definitions():
            got = oracle.mlp_raw(W, b, x)   # one (output) layer: sigmoid of the dot product
        for j in range(16):
            z = np.float32(math.fsum([float(b[0][j])] + [float(W[0][k, j]) * float(x16[k]) for k in range(64)]))
            ref = np.float32(1.0 / (1.0 + math.exp(-float(z))))
            assert got[j] == ref


# ---------------------------------------------------------------- the measurement
def _material_report(cfg, rows, dot=None, act=None, split=0):
    """Words + MLP outputs of `rows` of config `cfg` in the oracle mode (dot, act) vs the plain mode."""
    W, H, _ = synth.config_shape(cfg)
    om = oracle.Model(synth.model_blob(cfg))
    r0, r1 = rows
    saved = (oracle.get_dot_model(), int(L.o_get_act_model()))
    try:
        L.o_set_operand_model(split)
        if dot is not None:
            oracle.set_dot_model(*dot)
        if act is not None:
            oracle.set_act_model(act)
        w = om.decode_material(W, H, r0, r1)
        ep, col = om.mlp_outputs(W, H, r0, r1)
        oracle.set_dot_model(*saved[0])
        oracle.set_act_model(saved[1])
        with oracle.plain_definitions():
            pw = om.decode_material(W, H, r0, r1)
            pep, pcol = om.mlp_outputs(W, H, r0, r1)
    finally:
        oracle.set_dot_model(*saved[0])
        oracle.set_act_model(saved[1])
        L.o_set_operand_model(0)
    rep = compare_words(om.fmts, w, pw, pep, pcol)
    rep["endpoint_floats"] = float_stats(ep, pep)
    rep["colour_floats"] = float_stats(col, pcol)
    return rep


VARIANTS = {
    # name: (dot model, activation model); None = the pinned default
    "pinned (= CUDA path)": (None, None),
    "plain, sequential binary32 dot": ((1, 1, 100, 0), 1),
    "plain, binary32 libm activations": ((0, 16, 100, 0), 2),
}


@pytest.fixture(scope="module")
def reports():
    out = {}
    for cfg, rows in ((1, (0, 16)), (2, (0, 32))):
        for name, (dot, act) in VARIANTS.items():
            out[(cfg, name)] = _material_report(cfg, rows, dot, act)
    path = os.path.join(ROOT, "profiles", "faithfulness_cpu.json")
    try:
        with open(path, "w") as f:
            json.dump({f"C{c} {n}": r for (c, n), r in out.items()}, f, indent=1)
    except OSError:
        pass
    for (c, n), r in out.items():
        print(f"\nC{c} {n}: {r['mismatched']} of {r['words']} words differ "
              f"({r['excused']} excused, {r['unexcused']} unexcused); "
              + ", ".join(f"{k} {r[k][0]}/{r[k][1]}" for k in CLASSES)
              + f"; max rel endpoint {r['endpoint_floats']['max_rel']:.2e} colour {r['colour_floats']['max_rel']:.2e}")
    return out


@pytest.mark.parametrize("cfg", [1, 2])
def test_pinned_arithmetic_within_the_half_precision_floor(reports, cfg):
    """the pinned arithmetic (R9 v4 + R10) deviates from the plain definitions no more
    than other plain readings of the same half-precision network deviate from each other: its float
    deviation stays within twice the larger plain-variant deviation, and its mismatched / unexcused word
    counts within twice the larger plain variant's plus a Poisson allowance of 4 (sampling noise of rare
    counts).  An arithmetic bug (a dropped term, a wrong sign or constant) breaks this by orders of
    magnitude; the bounds are relative to measured plain variants, not to the kernel."""
    pin = reports[(cfg, "pinned (= CUDA path)")]
    others = [reports[(cfg, n)] for n in VARIANTS if not n.startswith("pinned")]
    for key in ("endpoint_floats", "colour_floats"):
        floor = max(o[key]["max_rel"] for o in others)
        assert pin[key]["max_rel"] <= 2 * floor + 1e-6, (key, pin[key]["max_rel"], floor)
        assert pin[key]["zero_violations"] == 0
    for key in ("mismatched", "unexcused"):
        floor = max(o[key] for o in others)
        assert pin[key] <= 2 * floor + 4, (key, pin[key], floor)


def test_contract_f_pinned_arithmetic_meets_the_literal_rule():
    """With binary32 activations (contract F of SURVEY §8.c.3: each MMA operand the split hi = RN16(a),
    lo = RN16(a - hi)) the pinned arithmetic -- R9 v4's exponential, R10's tensor-core summation order --
    meets north_star's rule LITERALLY against the plain definitions of the same contract: floats within
    1e-3 relative, zero unexcused words, excused words under 1e-4 of the blocks.  So the floor measured under
    the paper's half precision (contract H, test_pinned_arithmetic_within_the_half_precision_floor) is the
    contract's, not the pinned arithmetic's."""
    rep = _material_report(2, (0, 32), split=1)
    print(f"\nC2 rows 0-31, contract F, pinned vs plain: {rep['mismatched']} of {rep['words']} words differ "
          f"({rep['excused']} excused, {rep['unexcused']} unexcused); max rel endpoint "
          f"{rep['endpoint_floats']['max_rel']:.2e} colour {rep['colour_floats']['max_rel']:.2e}")
    assert rep["endpoint_floats"]["max_rel"] <= 1e-3 and rep["colour_floats"]["max_rel"] <= 1e-3
    assert rep["endpoint_floats"]["zero_violations"] == 0 and rep["colour_floats"]["zero_violations"] == 0
    assert rep["unexcused"] == 0
    assert rep["excused"] < 1e-4 * rep["blocks"]


def test_mismatch_classes_account_for_every_word(reports):
    for r in reports.values():
        assert sum(sum(r[c]) for c in CLASSES) == r["mismatched"] == r["excused"] + r["unexcused"]

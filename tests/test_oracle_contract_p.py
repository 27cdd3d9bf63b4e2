"""Pins of the oracle's contract P (-m "not gpu", R9-P): the hidden
selu evaluated in IEEE binary16 arithmetic, the most literal reading of "inference is executed in the
half-precision floating points".

What pins it (none of it re-derives the oracle's formula): the binary64 -> binary16 rounding against numpy's
(a library routine); every binary16 operation against exact rational arithmetic rounded by brute force over
the binary16 grid; the algorithm's exactness claims (integer t, Cody-Waite step, exponent insertion) checked
in exact arithmetic for every binary16 input; the result against the float64 libm selu within the error the
binary16 constants and roundings allow; special values.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle

L = oracle.lib()
LAM = 1.0507009873554804934
LAM_ALPHA = 1.0507009873554804934 * 1.6732632423543772848

# every finite binary16 value, ascending, with its bit pattern (brute-force rounding reference)
_bits = np.arange(0, 1 << 16, dtype=np.uint32).astype(np.uint16)
_vals = _bits.view(np.float16).astype(np.float64)
_fin = np.isfinite(_vals) & ~((_bits == 0x8000))      # -0 dropped: +0 represents zero in the grid
_order = np.argsort(_vals[_fin], kind="stable")
GRID_V = _vals[_fin][_order]
GRID_B = _bits[_fin][_order]
GRID_F = [Fraction(float(v)) for v in GRID_V]


def rn16_exact(x: Fraction) -> int:
    """Round a rational to binary16, nearest-even, by search over the binary16 grid (overflow -> inf)."""
    if x >= Fraction(65520):
        return 0x7C00
    if x <= Fraction(-65520):
        return 0xFC00
    i = int(np.searchsorted(GRID_V, float(x)))
    best = None
    for j in range(max(0, i - 2), min(len(GRID_F), i + 3)):
        d = abs(GRID_F[j] - x)
        key = (d, int(GRID_B[j]) & 1)             # ties: even mantissa (last bit 0)
        if best is None or key < best[0]:
            best = (key, int(GRID_B[j]))
    b = best[1]
    if b == 0 and x < 0:
        return 0x8000                              # a negative value rounding to zero keeps its sign
    return b


def f16(b: int) -> Fraction:
    return Fraction(float(np.uint16(b).view(np.float16)))


def test_f64_to_f16_matches_numpy():
    """o_f64_to_f16 = numpy's binary64 -> binary16 conversion (round to nearest even from the binary64 bits)
    on log-uniform values over the whole range (subnormals, overflow edge), every exact midpoint between
    adjacent binary16 values and its binary64 neighbours."""
    rng = np.random.default_rng(11)
    x = np.exp(rng.uniform(math.log(1e-9), math.log(7e4), 40000)) * rng.choice([-1.0, 1.0], 40000)
    mids = (GRID_V[1:] + GRID_V[:-1]) / 2
    mids = mids[np.isfinite(mids)]
    x = np.concatenate([x, mids, np.nextafter(mids, np.inf), np.nextafter(mids, -np.inf), [0.0, -0.0, 65519.99, 65520.0]])
    got = np.array([L.o_f64_to_f16(float(v)) for v in x], np.uint16)
    with np.errstate(over="ignore"):
        ref = x.astype(np.float16).view(np.uint16)
    assert np.array_equal(got, ref)


def _adversarial_triples():
    # products landing exactly on a binary16 midpoint, then nudged by the smallest addends
    out = [(0x4200, 0x5D56, 0x0001), (0x4200, 0x5D56, 0x8001), (0x4200, 0x5D56, 0x0000)]   # 3 * 341.5 = 1024.5
    out += [(0x3C01, 0x3C01, 0x8001), (0x7BFF, 0x3C00, 0x5000), (0x7BFF, 0x3C01, 0x0000)]  # overflow edge
    out += [(0x0001, 0x0001, 0x0000), (0x0400, 0x3800, 0x0000), (0x03FF, 0x4000, 0x8001)]  # subnormal results
    return out


def test_h16_ops_are_single_roundings():
    """o_h16_fma / mul / sub: the exact result (rational arithmetic) rounded ONCE to binary16, on random
    operands over the whole binary16 range and on adversarial midpoint / overflow / subnormal cases."""
    rng = np.random.default_rng(5)
    fin = GRID_B[np.abs(GRID_V) < 300]
    trip = [tuple(int(v) for v in rng.choice(fin, 3)) for _ in range(3000)] + _adversarial_triples()
    for a, b, c in trip:
        assert L.o_h16_fma(a, b, c) == rn16_exact(f16(a) * f16(b) + f16(c)), (hex(a), hex(b), hex(c))
        assert L.o_h16_mul(a, b) == rn16_exact(f16(a) * f16(b)), (hex(a), hex(b))
        assert L.o_h16_sub(a, c) == rn16_exact(f16(a) - f16(c)), (hex(a), hex(c))


NEG_H = [b for b in range(0x8001, 0xC900 + 1)]    # every negative binary16 from -2^-24 down to -10


def test_selu_half_exactness_claims():
    """R9-P's exactness claims, checked in exact arithmetic for every negative binary16 input h >= -10:
    t = RN16(h log2e16 + 1039) is an integer in [1025, 1039]; the Cody-Waite step h - n ln2hi is exact in
    binary16; S = lambda alpha16 2^n by exponent insertion is the exact product."""
    for hb in NEG_H:
        x = hb
        t = L.o_h16_fma(x, 0x3DC5, 0x640F)
        tv = f16(t)
        assert tv.denominator == 1 and 1025 <= tv <= 1039, hex(hb)
        n = int(tv) - 1039
        nf = L.o_h16_sub(t, 0x640F)
        assert f16(nf) == n
        g = L.o_h16_fma(nf, 0xB98C, x)
        assert f16(g) == f16(x) - n * Fraction(355, 512), hex(hb)        # ln2hi = 0.693359375 = 355/512
        assert abs(f16(g)) <= Fraction(37, 100)
        S = (0x3F08 + (n << 10)) & 0xFFFF
        assert f16(S) == f16(0x3F08) * Fraction(2) ** n


def _ulp_dist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    def lin(u):
        u = u.astype(np.int32)
        return np.where(u & 0x8000, -(u & 0x7FFF), u)
    return np.abs(lin(a) - lin(b))


def test_selu_half_accuracy_vs_libm():
    """Against the float64 libm selu rounded once to binary16 (the correctly rounded result): every binary16
    input within 2 ulp on the negative branch and 1 ulp on the positive branch.  The bound follows from the
    binary16 constants (lambda16, lambda alpha16 are 7.6e-5 / 1.6e-4 off: ~0.2 ulp), the rounding of u and
    of S - lambda alpha16 (<= 1/2 ulp each) and the final rounding; z = RN16(z) exactly here, so the input
    rounding of the contract (a further 1/2 ulp of z) is not part of this pin."""
    neg = np.array(NEG_H + [0x8000], np.uint16)
    got = np.array([L.o_selu_half(float(v)) for v in neg.view(np.float16).astype(np.float32)], np.uint16)
    ref = np.array([LAM_ALPHA * math.expm1(float(v)) for v in neg.view(np.float16).astype(np.float64)])
    assert _ulp_dist(got, ref.astype(np.float16).view(np.uint16)).max() <= 2
    pos = np.arange(0x0000, 0x7BFF, 37, dtype=np.uint32).astype(np.uint16)
    with np.errstate(over="ignore"):
        ref = (LAM * pos.view(np.float16).astype(np.float64)).astype(np.float16).view(np.uint16)
    got = np.array([L.o_selu_half(float(v)) for v in pos.view(np.float16).astype(np.float32)], np.uint16)
    assert _ulp_dist(got, ref).max() <= 1


@pytest.mark.parametrize("z,want", [(0.0, 0x0000), (-0.0, 0x0000), (-1e-30, 0x0000), (-100.0, 0xBF08),
                                    (-10.0, 0xBF08), (1e6, 0x7C00), (1.0, 0x3C34)])
def test_selu_half_special_values(z, want):
    """+0 / -0 / a negative value rounding to -0 give +0 (the negative branch at n = 0, u = 0); far below
    -10 the branch is -lambda alpha16; overflow of RN16(z) gives +inf on the positive branch."""
    assert L.o_selu_half(z) == want


def test_contract_p_mlp_uses_the_half_selu():
    """In act model 3 the MLP's hidden layers output binary16 values (the next layer's RN16 is the
    identity) and differ from contract H's; the sigmoid output layer is the pinned one of contract H."""
    rng = np.random.default_rng(3)
    W = [(rng.standard_normal((16, 64)) * 0.4).astype(np.float16), (rng.standard_normal((64, 8)) * 0.3).astype(np.float16)]
    b = [(rng.standard_normal(64) * 0.1).astype(np.float16), (rng.standard_normal(8) * 0.1).astype(np.float16)]
    x = rng.uniform(-1, 1, 16).astype(np.float32)
    h_out = oracle.mlp_raw(W, b, x)
    zs = np.linspace(-30, 30, 601).astype(np.float32)
    sig_h = [L.o_sigmoid(float(z)) for z in zs]
    with oracle.contract_p():
        p_out = oracle.mlp_raw(W, b, x)
        assert L.o_get_act_model() == 3
        assert [L.o_sigmoid(float(z)) for z in zs] == sig_h
        hid = [L.o_selu(float(z)) for z in zs]
        assert all(float(np.float32(v).astype(np.float16)) == v for v in hid)
    assert L.o_get_act_model() == 0
    assert not np.array_equal(h_out, p_out)
    assert np.max(np.abs(h_out - p_out)) < 2e-2

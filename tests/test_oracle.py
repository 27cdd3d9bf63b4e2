"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins (P:n = PAPER.md line n, S:n = SPEC.md line n)
and what it is pinned against: a value the paper prints, a closed form, an
independent library routine (numpy, torch float64, math.fsum, Pillow), or brute
force.  None of these tests compares the oracle with itself or with the CUDA path.
"""
import io
import math
import os
import struct

import numpy as np
import pytest
import torch

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
L = oracle.lib()


def _golden_kv(name):
    kv = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if "=" in line:
            k, v = line.split("=", 1)
            kv[k.strip()] = v.strip()
    return kv


# ---------------------------------------------------------------- fp16
def test_f16_to_f32_all_codes_vs_numpy():
    h = np.arange(65536, dtype=np.uint16)
    ref = h.view(np.float16).astype(np.float32)
    got = np.array([L.o_f16_to_f32(int(x)) for x in h], np.float32)
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin].view(np.uint32), ref[fin].view(np.uint32))
    assert np.all(np.isnan(got[np.isnan(ref)]))


def test_f32_to_f16_exhaustive_vs_numpy():
    """Every binary32 value with |x| in [2^-26, 2^17) (all binary16 subnormal, normal and overflow
    binades, both signs) converts exactly as numpy's IEEE round-to-nearest-even."""
    lo = np.float32(2.0 ** -26).view(np.uint32)
    hi = np.float32(2.0 ** 17).view(np.uint32)
    step = 1 << 24
    for start in range(int(lo), int(hi), step):
        bits = np.arange(start, min(start + step, int(hi)), dtype=np.uint32)
        for sgn in (0, 0x80000000):
            x = (bits | np.uint32(sgn)).view(np.float32)
            with np.errstate(over="ignore"):
                ref = x.astype(np.float16).view(np.uint16)
            assert np.array_equal(oracle.f32_to_f16(x), ref), hex(start)


def test_f32_to_f16_round_nearest_even_vs_numpy():
    rng = np.random.default_rng(1)
    x = np.concatenate([
        rng.standard_normal(200000).astype(np.float32) * np.float32(3),
        (rng.random(50000) * 1e-4).astype(np.float32),          # subnormal range
        (rng.random(20000) * 70000).astype(np.float32),          # overflow edge
        np.array([0.0, -0.0, 65504, 65519.99, 65520, 2 ** -24, 2 ** -25, 3 * 2 ** -26, 2 ** -14], np.float32),
    ])
    # halfway cases: odd multiples of half a binary16 quantum
    halves = (np.arange(1, 4000, 2) * 2.0 ** -12).astype(np.float32)
    x = np.concatenate([x, halves, -halves])
    with np.errstate(over="ignore"):
        ref = x.astype(np.float16).view(np.uint16)
    got = np.array([L.o_f32_to_f16(float(v)) for v in x], np.uint16)
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------- Eq.2 dequantization
def test_dequant_eq2_single_rounding():
    for s in (np.float32(0.0078125), np.float32(0.00731), np.float32(0.0111)):
        for z in (0, 100, 128, 255):
            q = np.arange(256)
            ref = (np.float64(s) * (q - z)).astype(np.float32)   # exact product, one RN
            got = np.array([L.o_dequant(int(v), float(s), z) for v in q], np.float32)
            assert np.array_equal(got, ref)


# ---------------------------------------------------------------- pinned exp (R9), selu / sigmoid
# The accuracy bound of the pinned exponential is fixed by the paper, not by the implementation:
# the hidden activations are stored in binary16, so E and the selu branch must stay
# within 1/16 of a binary16 ulp (relative 2^-15) of the exact function everywhere, including the
# selu branch as z -> 0^- (no cancellation: its binary16 result must not depend on how E is built).
# These bounds do not move when the kernel changes.
BIN16_ULP_16 = 2.0 ** -15
SELU_LAMBDA, SELU_ALPHA = 1.0507009873554804934, 1.6732632423543772848


def test_exp_accuracy_vs_libm():
    """R9: E(x) within 2^-15 relative of e^x on the whole clamp range (libm exp in float64)."""
    assert L.o_exp(0.0) == 1.0
    assert L.o_exp_max_relerr(-80.0, 80.0, 100003, 0) < BIN16_ULP_16
    assert L.o_exp_max_relerr(-10.0, 10.0, 10007, 0) < BIN16_ULP_16


def test_selu_branch_relative_error_near_zero():
    """R9: lambda alpha (e^z - 1) within 2^-15 RELATIVE of the exact value (libm expm1, exact
    constants) for every z in (-80, 0), densely down to z = -1e-38: no cancellation as z -> 0^-."""
    z = -np.concatenate([np.geomspace(1e-38, 80, 60001), np.linspace(1e-4, 20, 40001)]).astype(np.float32)
    got = np.array([L.o_selu(float(v)) for v in z], np.float64)
    ref = SELU_LAMBDA * SELU_ALPHA * np.expm1(z.astype(np.float64))
    assert np.max(np.abs(got - ref) / np.abs(ref)) < BIN16_ULP_16
    la = float(np.float32(SELU_LAMBDA * SELU_ALPHA))
    assert np.all(got <= 0.0) and np.all(got >= -la)                # range of the branch
    assert np.all(np.diff(got[:60001]) <= 0.0)                     # non-increasing as z decreases
    assert L.o_exp_max_relerr(-80.0, -1e-30, 20011, 1) < BIN16_ULP_16


def test_selu_sigmoid_vs_torch_float64():
    z = np.concatenate([np.linspace(-30, 30, 20001), np.geomspace(1e-8, 1, 2000) * -1]).astype(np.float32)
    zt = torch.from_numpy(z.astype(np.float64))
    ref_selu = torch.nn.functional.selu(zt).numpy()
    ref_sig = torch.sigmoid(zt).numpy()
    got_selu = np.array([L.o_selu(float(v)) for v in z])
    got_sig = np.array([L.o_sigmoid(float(v)) for v in z])
    nz = ref_selu != 0
    assert np.all(got_selu[~nz] == 0.0)
    assert np.max(np.abs(got_selu[nz] - ref_selu[nz]) / np.abs(ref_selu[nz])) < BIN16_ULP_16
    assert np.max(np.abs(got_sig - ref_sig) / ref_sig) < BIN16_ULP_16
    assert L.o_selu(0.0) == 0.0 and L.o_sigmoid(0.0) == 0.5
    assert L.o_sigmoid(1e30) == 1.0 and 0.0 <= L.o_sigmoid(-1e30) < 1e-30


# ---------------------------------------------------------------- exact fused summation (R10)
def _rand_f16(rng, n, lo=-6, hi=6):
    mag = np.exp2(rng.uniform(lo, hi, n)) * rng.choice([-1, 1], n)
    return mag.astype(np.float16)


def test_fused_sum_exact_then_rn_vs_fsum():
    """With p large the fused sum is the exact sum rounded once (RN) to binary32."""
    rng = np.random.default_rng(2)
    for _ in range(3000):
        n = int(rng.integers(1, 65))
        a, b = _rand_f16(rng, n), _rand_f16(rng, n)
        acc = np.float32(rng.standard_normal() * 4)
        exact = math.fsum([float(acc)] + [float(x) * float(y) for x, y in zip(a, b)])  # exact: span < 53 bits
        ref = np.float32(exact)
        got = oracle.fused_sum(float(acc), a, b, 100, 0)
        assert got == ref, (got, ref)


def test_fused_sum_truncation_bound():
    """Truncating below 2^(lead-p) moves the sum by < n * 2^(lead-p) before the final rounding."""
    rng = np.random.default_rng(3)
    for p in (24, 25, 26, 28):
        for _ in range(1000):
            n = 16
            a, b = _rand_f16(rng, n, -12, 6), _rand_f16(rng, n, -12, 6)
            prods = [float(x) * float(y) for x, y in zip(a, b)]
            exact = math.fsum(prods)
            lead = max(math.frexp(v)[1] - 1 for v in prods if v != 0)
            bound = (n + 1) * 2.0 ** (lead - p) + abs(exact) * 2.0 ** -23
            for rm in (0, 1):
                got = oracle.fused_sum(None, a, b, p, rm)
                assert abs(got - exact) <= bound


def test_fused_sum_representable_is_exact():
    """Sums whose terms all fit inside the p-bit window are exact in every model."""
    rng = np.random.default_rng(4)
    for _ in range(500):
        a = (rng.integers(-64, 64, 16)).astype(np.float16)       # small integers
        b = (rng.integers(-64, 64, 16)).astype(np.float16)
        exact = float(np.dot(a.astype(np.int64), b.astype(np.int64)))
        for p in (24, 30, 100):
            for rm in (0, 1):
                assert oracle.fused_sum(None, a, b, p, rm) == exact


# ---------------------------------------------------------------- MLP
def _torch_mlp(weights, biases, x):
    """float64 torch reference with fp16 rounding of every layer input."""
    a = torch.from_numpy(np.asarray(x, np.float64))
    for li, (w, b) in enumerate(zip(weights, biases)):
        a16 = a.to(torch.float16).to(torch.float64)
        z = a16 @ torch.from_numpy(w.astype(np.float64)) + torch.from_numpy(b.astype(np.float64))
        a = torch.nn.functional.selu(z) if li + 1 < len(weights) else torch.sigmoid(z)
    return a.numpy()


def test_mlp_single_layer_vs_torch_float64():
    """One layer = sigmoid(b + x16 @ W): pins the operand rounding, the Dot and the orientation of W."""
    rng = np.random.default_rng(5)
    orig = oracle.get_dot_model()
    for mode in ((0, 16, 100, 0), orig):
        oracle.set_dot_model(*mode)
        for _ in range(50):
            i, o = int(rng.integers(1, 65)), int(rng.integers(1, 33))
            w = (rng.standard_normal((i, o)) * np.sqrt(2 / i)).astype(np.float16)
            b = rng.uniform(-0.1, 0.1, o).astype(np.float16)
            x = rng.standard_normal(i).astype(np.float32)
            got = oracle.mlp_raw([w], [b], x)
            ref = _torch_mlp([w], [b], x)
            assert np.max(np.abs(got - ref) / ref) < 1e-5   # R9: E within 7.3e-6 (relative)
    oracle.set_dot_model(*orig)


def test_mlp_paper_architecture_vs_torch_float64():
    """16 -> 64 -> 64 -> 64 -> 9 with selu/sigmoid against torch float64 with binary16 layer
    inputs.  The plain-definition mode agrees to 1e-6 relative on every sample (it differs from torch only
    by its binary32 roundings): this pins the architecture, the operand rounding, the weight orientation and
    the selu constants tightly.  The pinned mode (R9, R10) agrees to 1e-5 on at least 90% of the samples; on
    the rest a one-ulp difference of a pre-activation flipped a binary16 rounding, bounded by 2e-3."""
    rng = np.random.default_rng(6)
    close = 0
    n = 60
    for _ in range(n):
        dims = [16, 64, 64, 64, 9]
        ws = [(rng.standard_normal((i, o)) * np.sqrt(2 / i)).astype(np.float16) for i, o in zip(dims[:-1], dims[1:])]
        bs = [rng.uniform(-0.1, 0.1, o).astype(np.float16) for o in dims[1:]]
        x = rng.uniform(-1, 1, 16).astype(np.float32)
        ref = _torch_mlp(ws, bs, x)
        with oracle.plain_definitions():
            plain = oracle.mlp_raw(ws, bs, x)
        assert np.max(np.abs(plain - ref) / np.abs(ref)) < 1e-6
        got = oracle.mlp_raw(ws, bs, x)
        assert np.max(np.abs(got - ref)) < 2e-3
        close += np.max(np.abs(got - ref) / np.abs(ref)) < 1e-5
    assert close >= 0.9 * n, close


def test_mlp_zero_weights_gives_half():
    w = [np.zeros((16, 64), np.float16), np.zeros((64, 64), np.float16), np.zeros((64, 5), np.float16)]
    b = [np.zeros(64, np.float16), np.zeros(64, np.float16), np.zeros(5, np.float16)]
    assert np.all(oracle.mlp_raw(w, b, np.ones(16, np.float32)) == 0.5)


# ---------------------------------------------------------------- grid encoding
def _grid_model(res_list, codes_fn, s=0.01, z=128):
    sp = synth.ModelSpec([synth.BC1], hidden=16, block_levels=len(res_list), block_coarsest=res_list[0],
                         texel_levels=len(res_list), texel_coarsest=res_list[0])
    m = synth.random_model(sp, 1)
    m.block_grid = [(np.float32(s), np.int32(z), codes_fn(r)) for r in sp.level_res("block")]
    m.texel_grid = [(np.float32(s), np.int32(z), codes_fn(r)) for r in sp.level_res("texel")]
    return m


def test_grid_encode_vs_torch_grid_sample():
    """Vertex-centred bilinear lookup (R1) = grid_sample(align_corners=True) in float64."""
    rng = np.random.default_rng(7)
    sp = synth.ModelSpec([synth.BC1, synth.BC4])
    sp.texel_levels = 4
    sp.block_levels = 3
    m = synth.random_model(sp, 11)
    om = oracle.Model(synth.serialize(m))
    pts = rng.random((300, 2)).astype(np.float32)
    for which, grid in ((0, m.block_grid), (1, m.texel_grid)):
        got = np.stack([om.grid_encode(which, float(p), float(q)) for p, q in pts])
        for l, (s, z, codes) in enumerate(grid):
            vals = float(s) * (codes.astype(np.float64) - float(z))            # Eq.2, [res][res][F]
            inp = torch.from_numpy(vals.transpose(2, 0, 1)[None])               # N C H W
            g = torch.from_numpy((pts.astype(np.float64) * 2 - 1)[None, :, None, :])  # (x=p, y=q)
            ref = torch.nn.functional.grid_sample(inp, g, mode="bilinear", align_corners=True)[0, :, :, 0].T.numpy()
            assert np.max(np.abs(got[:, 2 * l:2 * l + 2] - ref)) < 2e-5, (which, l)


def test_grid_encode_reproduces_affine_field_and_centre():
    """Bilinear interpolation reproduces an affine vertex field; cell centre = mean of 4."""
    def affine(r):
        j, i = np.meshgrid(np.arange(r), np.arange(r), indexing="ij")
        a = 30 + (i * 150) // (r - 1)            # integer codes, exactly affine only if divisible
        b = 40 + (j * 120) // (r - 1)
        return np.stack([a, b], -1).astype(np.uint8)
    m = _grid_model([16], affine, s=0.5, z=0)
    # res 16: (r-1)=15 divides 150 and 120, so codes are exactly affine in i and j
    om = oracle.Model(synth.serialize(m))
    rng = np.random.default_rng(8)
    for p, q in rng.random((200, 2)).astype(np.float32):
        X = np.float32(p) * np.float32(15)
        Y = np.float32(q) * np.float32(15)
        ref = [0.5 * (30 + 10 * float(X)), 0.5 * (40 + 8 * float(Y))]
        got = om.grid_encode(1, float(p), float(q))
        assert abs(got[0] - ref[0]) < 1e-4 and abs(got[1] - ref[1]) < 1e-4
    # cell centre: X = 0.5 exactly when p = 0.5/15 ... use p with X exactly i+0.5
    rcodes = np.random.default_rng(9).integers(0, 256, (16, 16, 2)).astype(np.uint8)
    m2 = _grid_model([16], lambda r: rcodes, s=1.0, z=0)
    om2 = oracle.Model(synth.serialize(m2))
    p = np.float32(np.float32(7.5) / np.float32(15))
    X = p * np.float32(15)
    if X == np.float32(7.5):
        got = om2.grid_encode(1, float(p), float(p))
        ref = rcodes[7:9, 7:9].astype(np.float64).mean(axis=(0, 1))
        assert np.allclose(got, ref, atol=1e-4)


# ---------------------------------------------------------------- BC formats (Eq.7/8)
MAP1 = [0, 2, 3, 1]


def test_bc_layout_goldens():
    for line in open(os.path.join(GOLDEN, "bc_layout.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        name, fmt, word, texels = [x.strip() for x in line.split("|")]
        fmt = int(fmt)
        word = int(word.replace("_", ""), 16)
        val = eval(texels.split("*")[1])
        got = oracle.decode_block(word, fmt)
        exp = np.tile(np.array(val, np.float32), (16, 1)) if fmt == 1 else np.full(16, val, np.float32)
        assert np.array_equal(got, exp), name


def test_code_maps_golden_vs_decoder():
    kv = _golden_kv("maps.txt")
    maps = {k: [int(x) for x in v.split()] for k, v in kv.items()}
    # BC1: decode each stored code and match it with the linear palette entry
    e0, e1 = 0xF800, 0x001F
    pal = oracle.palette_bc1([1, 0, 0], [0, 0, 1])
    for n, code in enumerate(maps["bc1"]):
        blk = e0 | (e1 << 16) | (sum(code << (2 * i) for i in range(16)) << 32)
        assert np.array_equal(oracle.decode_block(blk, 1)[0], pal[n])
    for (E0, E1), key in (((200, 50), "bc4_e0_gt_e1"), ((50, 200), "bc4_e0_le_e1")):
        pal = oracle.palette_bc4(E0, E1)
        for n, code in enumerate(maps[key]):
            blk = E0 | (E1 << 8) | (sum(code << (3 * i) for i in range(16)) << 16)
            assert oracle.decode_block(blk, 4)[0] == pal[n]


def _dds(fourcc, w, h, payload):
    hdr = struct.pack("<4sIIIIIII44s", b"DDS ", 124, 0x1 | 0x2 | 0x4 | 0x1000 | 0x80000, h, w,
                      len(payload), 0, 1, b"\0" * 44)
    hdr += struct.pack("<II4sIIIII", 32, 0x4, fourcc, 0, 0, 0, 0, 0)          # DDS_PIXELFORMAT
    hdr += struct.pack("<IIIII", 0x1000, 0, 0, 0, 0)                         # caps
    assert len(hdr) == 128
    return hdr + payload


def test_decoder_cross_check_with_pillow():
    """Pillow's independent DXT1/ATI1 decoder agrees within +-2 LSB (it bit-replicates RGB565 and
    interpolates in integers).  A wrong bit order or code map is off by tens of LSBs."""
    from PIL import Image
    rng = np.random.default_rng(10)
    nb = 64
    blocks1 = []
    for _ in range(nb):
        c0, c1 = sorted(rng.integers(0, 65536, 2).tolist(), reverse=True)
        if c0 == c1:
            c1 = max(0, c0 - 1)
        blocks1.append(c0 | (c1 << 16) | (int(rng.integers(0, 2 ** 32)) << 32))
    blocks4 = [int(rng.integers(0, 2 ** 63)) | (int(rng.integers(0, 2)) << 63) for _ in range(nb)]
    W, H = 4 * 8, 4 * 8
    for fmt, blocks, cc in ((1, blocks1, b"DXT1"), (4, blocks4, b"ATI1")):
        arr = np.array(blocks, np.uint64)
        img = Image.open(io.BytesIO(_dds(cc, W, H, arr.tobytes())))
        img.load()
        pil = np.asarray(img).astype(np.float64)
        ours = oracle.decode_bc(arr, fmt, W, H).astype(np.float64) * 255
        if fmt == 1:
            pil = pil[..., :3]
        else:
            pil = pil.reshape(H, W, -1)[..., :1]
        assert np.max(np.abs(pil - ours)) <= 2.0 + 1e-9, fmt


def test_palette_goldens():
    for line in open(os.path.join(GOLDEN, "palettes.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        fmt, ee, vals, _ = [x.strip() for x in line.split("|")]
        E0, E1 = [int(x, 0) for x in ee.split()]
        exp = np.array([float(v) for v in vals.split()])
        if int(fmt) == 4:
            got = oracle.palette_bc4(E0, E1)
        else:
            e0, e1 = np.zeros(3, np.float32), np.zeros(3, np.float32)
            L.o_expand565(E0, e0.ctypes.data)
            L.o_expand565(E1, e1.ctypes.data)
            got = oracle.palette_bc1(e0, e1)[:, 0]
        assert np.max(np.abs(got - exp)) < 1e-6


def test_eq8_identities_and_endpoints_all_pairs():
    """Eq.8 first/third cases give exactly 0 and 1; n=0 / n=7 reproduce e0 / e1 in mode e0>e1;
    interior entries equal (1-w)e0 + w e1 to within one rounding."""
    for E0 in range(256):
        for E1 in range(256):
            pal = oracle.palette_bc4(E0, E1)
            e0, e1 = np.float32(E0) / np.float32(255), np.float32(E1) / np.float32(255)
            if E0 > E1:
                assert pal[0] == e0 and pal[7] == e1
                w = np.arange(8) / 7
            else:
                assert pal[0] == 0.0 and pal[7] == 1.0
                assert pal[1] == e0 and pal[6] == e1
                w = np.concatenate([[0], np.arange(6) / 5, [0]])
            ref = (1 - w) * float(e0) + w * float(e1)
            sl = slice(0, 8) if E0 > E1 else slice(1, 7)
            assert np.max(np.abs(pal[sl] - ref[sl])) < 2e-7


def test_endpoint_quantizer_round_trip():
    """R11: E = floor(e*(2^b-1)+1/2) inverts the UNORM expansion for every code (exhaustive)."""
    for k in range(256):
        assert L.o_unorm8(float(np.float32(k) / np.float32(255))) == k
    e = np.zeros(3, np.float32)
    for c in range(65536):
        L.o_expand565(c, e.ctypes.data)
        assert L.o_rgb565(e.ctypes.data) == c


def test_index_selection_is_bruteforce_nearest():
    """Eq.9-10: chosen n minimises the exact distance to the palette (float64 brute force)."""
    rng = np.random.default_rng(12)
    for _ in range(2000):
        pal = rng.random((4, 3)).astype(np.float32)
        c = rng.random(3).astype(np.float32)
        n = L.o_argmin_bc1(c.ctypes.data, pal.ctypes.data)
        d = np.sum((c.astype(np.float64) - pal.astype(np.float64)) ** 2, axis=1)
        assert d[n] <= d.min() + 1e-6
        E0, E1 = (int(x) for x in rng.integers(0, 256, 2))
        p4 = oracle.palette_bc4(E0, E1)
        v = np.float32(rng.random())
        n4 = L.o_argmin_bc4(float(v), p4.ctypes.data)
        d4 = np.abs(float(v) - p4.astype(np.float64))
        assert d4[n4] <= d4.min() + 1e-7
        if np.sum(d4 == d4.min()) > 1:
            assert n4 == int(np.argmin(d4))          # ties -> lowest linear n (R15)


def test_decode_of_encode_is_palette_of_argmin():
    rng = np.random.default_rng(13)
    for _ in range(500):
        ep = rng.random(6).astype(np.float32)
        tx = rng.random((16, 3)).astype(np.float32)
        w = oracle.encode_bc1(ep, tx)
        c0, c1 = w & 0xFFFF, (w >> 16) & 0xFFFF
        assert c0 > c1 or (c0 == c1 and (w >> 32) == 0)           # 4-colour mode (R12)
        dec = oracle.decode_block(w, 1)
        if c0 != c1:
            e0, e1 = np.zeros(3, np.float32), np.zeros(3, np.float32)
            L.o_expand565(c0, e0.ctypes.data)
            L.o_expand565(c1, e1.ctypes.data)
            pal = oracle.palette_bc1(e0, e1)
            for i in range(16):
                d = np.sum((tx[i].astype(np.float64) - pal.astype(np.float64)) ** 2, axis=1)
                assert np.sum((tx[i] - dec[i]) ** 2) <= d.min() + 1e-6
        ep4 = rng.random(2).astype(np.float32)
        t4 = rng.random(16).astype(np.float32)
        w4 = oracle.encode_bc4(ep4, t4)
        pal4 = oracle.palette_bc4(w4 & 255, (w4 >> 8) & 255)
        dec4 = oracle.decode_block(w4, 4)
        for i in range(16):
            assert abs(float(t4[i]) - float(dec4[i])) <= np.min(np.abs(float(t4[i]) - pal4.astype(np.float64))) + 1e-7


def test_bc4_bruteforce_optimum_bounds_ntbc_encoding():
    """Exhaustive BC4 search over all 65,536 endpoint pairs: the NTBC block (any predicted
    endpoints) can never beat it, and two-level blocks are encoded exactly."""
    rng = np.random.default_rng(14)
    for _ in range(4):
        tx = rng.random(16).astype(np.float32)
        blk, best = oracle.bruteforce_bc4(tx)
        assert abs(oracle.block_sq_error(blk, 4, tx) - best) < 1e-9
        for _ in range(20):
            w = oracle.encode_bc4(rng.random(2).astype(np.float32), tx)
            assert oracle.block_sq_error(w, 4, tx) >= best - 1e-12
    # a block made of two representable values (in mode e0>e1) has optimal error 0 and NTBC finds it
    a, b = np.float32(200) / np.float32(255), np.float32(60) / np.float32(255)
    tx = np.where(rng.random(16) < 0.5, a, b).astype(np.float32)
    blk, best = oracle.bruteforce_bc4(tx)
    assert best == 0.0
    assert oracle.block_sq_error(oracle.encode_bc4(np.array([a, b], np.float32), tx), 4, tx) == 0.0


def test_bc1_two_colour_block_is_exact():
    rng = np.random.default_rng(15)
    for _ in range(200):
        c = sorted(rng.integers(0, 65536, 2).tolist(), reverse=True)
        if c[0] == c[1]:
            continue
        e = np.zeros((2, 3), np.float32)
        for i in range(2):
            L.o_expand565(c[i], e[i].ctypes.data)
        tx = e[rng.integers(0, 2, 16)]
        w = oracle.encode_bc1(e.reshape(-1), tx)
        assert oracle.block_sq_error(w, 1, tx) == 0.0


# ---------------------------------------------------------------- end to end
def _closed_form_blob(fmt):
    big = 65504.0
    if fmt == synth.BC1:
        spec = synth.ModelSpec([synth.BC1], hidden=16, block_levels=2, block_coarsest=8, texel_levels=2, texel_coarsest=16)
        ep_b = [big, -big, -big, -big, -big, big]
        co_b = [math.log(2.0), -big, -math.log(2.0)]
    else:
        spec = synth.ModelSpec([synth.BC4], hidden=16, block_levels=2, block_coarsest=8, texel_levels=2, texel_coarsest=16)
        ep_b = [1.291, -1.411]
        co_b = [0.129]
    return synth.serialize(synth.closed_form_model(spec, ep_b, co_b))


def test_closed_form_end_to_end_golden():
    kv = _golden_kv("closed_form.txt")
    for fmt, key in ((synth.BC1, "bc1_word"), (synth.BC4, "bc4_word")):
        m = oracle.Model(_closed_form_blob(fmt))
        out = m.decode_material(16, 8)
        assert np.all(out == np.uint64(int(kv[key], 16))), (key, hex(int(out.flat[0])))


def test_pack_of_mlp_outputs_equals_decode_material():
    m = oracle.Model(synth.model_blob(1))
    ep, col = m.mlp_outputs(64, 64)
    assert np.array_equal(oracle.pack(m.fmts, ep, col, 64, 64), m.decode_material(64, 64))
    assert np.array_equal(m.decode_material(64, 64, 3, 9), m.decode_material(64, 64)[:, 3:9])


def test_model_parse_rejects_bad_blobs():
    blob = synth.model_blob(1)
    for bad in (b"XTBC" + blob[4:], blob[:500], blob[:4] + struct.pack("<I", 2) + blob[8:]):
        with pytest.raises(ValueError):
            oracle.Model(bad)


# ---------------------------------------------------------------- storage and PSNR
def test_storage_arithmetic_reproduces_paper_numbers():
    kv = _golden_kv("storage.txt")
    sb = lambda bl, tl, ne, nc, bias=1: L.o_storage_bytes(bl, 16, tl, 16, 2, 64, 3, ne, nc, bias)
    # grid payload alone (no MLP): hidden=0 layers of width 0 contribute 2*(in*out)=0 with out=0
    grids_only = L.o_storage_bytes(7, 16, 8, 16, 2, 0, 0, 0, 0, 0) - 0
    assert grids_only == int(kv["texel_grid_bytes"]) + int(kv["block_grid_bytes"])
    ag = sb(7, 8, 6 * 2 + 2 * 4, 3 * 2 + 4)            # aggressive: 2 BC1 + 4 BC4
    cs = sb(7, 8, 6 * 2, 3 * 2) + sb(7, 8, 2 * 4, 4)   # conservative pair
    assert round(ag / 2 ** 20, 2) == float(kv["aggressive_MiB"])
    assert round(cs / 2 ** 20, 2) == float(kv["conservative_MiB"])
    assert 1024 * 1024 * 8 / 2 ** 20 == float(kv["bc_texture_4k_MiB"])


def test_psnr_uniform_error_closed_form():
    rng = np.random.default_rng(16)
    a = rng.random(4096).astype(np.float32) * 0.5
    for eps in (0.1, 0.01, 1 / 255):
        b = a + np.float32(eps)
        ref = 20 * math.log10(1 / float(np.float32(eps)))
        assert abs(oracle.psnr(a, b) - ref) < 1e-3


# ---------------------------------------------------------------- naive approach
def test_naive_weight_quantization_spec_examples():
    """SPEC quantize_weight examples: 0.34 -> n=1 (nearest of {0, 1/3, 2/3, 1}); 0 -> 0; BC4 E0 > E1 with
    w = 0.5 exactly between 3/7 and 4/7 -> the lower n (3)."""
    assert oracle.quantize_weight(0.34, synth.BC1) == 1
    assert oracle.quantize_weight(0.0, synth.BC1) == 0
    assert oracle.quantize_weight(1.0, synth.BC1) == 3
    assert oracle.quantize_weight(0.5, synth.BC4, True) == 3
    # 6-value mode: the weights (n-1)/5 of entries 1..6; the constant entries 0 and 7 are never chosen
    ws = np.linspace(0.0, 1.0, 2001)
    ns = {oracle.quantize_weight(float(w), synth.BC4, False) for w in ws}
    assert ns == {1, 2, 3, 4, 5, 6}
    assert oracle.quantize_weight(0.0, synth.BC4, False) == 1 and oracle.quantize_weight(1.0, synth.BC4, False) == 6


def test_naive_encoding_decodes_to_nearest_palette_colour_of_the_weighted_mix():
    """Independent pin of the naive encoders (Eq.7/8): every palette entry lies on the segment
    between the quantized endpoints and is ordered by its weight, so the decoded texel of a naive block
    must be the palette colour nearest to the weighted mix (1-w) e0 + w e1 of the endpoints in the
    PREDICTED order -- which also pins the BC1 index remap when the 4-colour rule swaps them.  Weights
    are drawn away from the midpoints between palette weights, where fp32 rounding decides ties."""
    rng = np.random.default_rng(7)
    checked_swap = 0
    for _ in range(300):
        ep = rng.uniform(0, 1, 6).astype(np.float32)
        c0, c1 = oracle.rgb565(ep[:3]), oracle.rgb565(ep[3:])
        if c0 == c1:
            continue
        e0, e1 = oracle.expand565(c0), oracle.expand565(c1)   # quantized endpoints, predicted order
        ws = rng.uniform(0, 1, 16).astype(np.float32)
        mid = np.array([1 / 6, 1 / 2, 5 / 6])
        ws = np.where(np.min(np.abs(ws[:, None] - mid[None, :]), axis=1) < 1e-3, 0.25, ws).astype(np.float32)
        blk = oracle.encode_bc1_naive(ep, ws)
        dec = oracle.decode_block(blk, synth.BC1).reshape(16, 3)
        want = [(1 - w) * e0 + w * e1 for w in ws.astype(np.float64)]
        pal = [(1 - t) * e0 + t * e1 for t in (0, 1 / 3, 2 / 3, 1)]
        for i in range(16):
            best = min(pal, key=lambda c: np.sum((c - want[i]) ** 2))
            assert np.allclose(dec[i], best, atol=1e-6), (i, ws[i], c0 < c1)
        checked_swap += c0 < c1
    assert checked_swap > 50
    for mode8 in (True, False):
        for _ in range(200):
            E = sorted(rng.choice(256, 2, replace=False))
            E0, E1 = (E[1], E[0]) if mode8 else (E[0], E[1])
            ep = np.array([E0 / 255, E1 / 255], np.float32)
            ws = rng.uniform(0, 1, 16).astype(np.float32)
            steps = np.arange(7) / 7 if mode8 else np.arange(5) / 5
            mids = (steps + (1 / 14 if mode8 else 1 / 10))
            ws = np.where(np.min(np.abs(ws[:, None] - mids[None, :]), axis=1) < 1e-3, 0.02, ws).astype(np.float32)
            blk = oracle.encode_bc4_naive(ep, ws)
            dec = oracle.decode_block(blk, synth.BC4)
            e0, e1 = E0 / 255, E1 / 255
            cand = [(1 - n / 7) * e0 + n / 7 * e1 for n in range(8)] if mode8 else \
                   [(1 - n / 5) * e0 + n / 5 * e1 for n in range(6)]
            for i in range(16):
                want = (1 - float(ws[i])) * e0 + float(ws[i]) * e1
                assert abs(dec[i] - min(cand, key=lambda c: abs(c - want))) < 1e-6


def test_naive_model_container_and_material():
    """The variant flag round-trips through the container; a naive model's texel net has one output
    per texture and decode_material equals the naive encoders applied to mlp_outputs."""
    for cfg in (7, 8):
        m = oracle.Model(synth.model_blob(cfg))
        assert m.naive and m.n_c == m.n_tex
    m = oracle.Model(synth.model_blob(8))
    W, H, _ = synth.config_shape(8)
    words = m.decode_material(W, H)
    ep, w = m.mlp_outputs(W, H)
    eo = 0
    for k, f in enumerate(m.fmts):
        for by in (0, 7, H // 4 - 1):
            for bx in (0, 5, W // 4 - 1):
                ws = np.array([w[4 * by + i // 4, 4 * bx + i % 4, k] for i in range(16)], np.float32)
                e = ep[by, bx, eo:eo + (6 if f == synth.BC1 else 2)]
                enc = oracle.encode_bc1_naive(e, ws) if f == synth.BC1 else oracle.encode_bc4_naive(e, ws)
                assert words[k, by, bx] == np.uint64(enc)
        eo += 6 if f == synth.BC1 else 2


# ---------------------------------------------------------------- reference encoder
def _codes(blk, fmt):
    return [(blk >> (32 + 2 * i)) & 3 for i in range(16)] if fmt == synth.BC1 else \
           [(blk >> (16 + 3 * i)) & 7 for i in range(16)]


def _with_code(blk, fmt, i, code):
    sh, m = (32 + 2 * i, 3) if fmt == synth.BC1 else (16 + 3 * i, 7)
    return (blk & ~(m << sh)) | (code << sh)


def test_ref_encoder_spec_examples():
    # constant BC4 block at 0.5: decoded error per texel <= 1/510 (quantization bound)
    blk = oracle.encode_ref_block(np.full(16, 0.5, np.float32), synth.BC4)
    assert np.all(np.abs(oracle.decode_block(blk, synth.BC4) - 0.5) <= 1 / 510 + 1e-7)
    # a block with exact 0 and 1 texels: the 6-value mode (E0 <= E1) represents both exactly and wins
    rng = np.random.default_rng(3)
    for _ in range(50):
        t = rng.uniform(0.3, 0.7, 16).astype(np.float32)
        t[rng.choice(16, 2, replace=False)] = [0.0, 1.0]
        blk = oracle.encode_ref_block(t, synth.BC4)
        assert (blk & 0xFF) <= ((blk >> 8) & 0xFF)
        dec = oracle.decode_block(blk, synth.BC4)
        assert np.all(dec[t == 0.0] == 0.0) and np.all(dec[t == 1.0] == 1.0)
    # degenerate BC1 block (all texels one colour): c0 == c1, all codes 0, within half a 565 step
    c = np.array([0.3, 0.6, 0.9], np.float32)
    blk = oracle.encode_ref_block(np.tile(c, (16, 1)), synth.BC1)
    assert (blk & 0xFFFF) == ((blk >> 16) & 0xFFFF) and (blk >> 32) == 0
    assert np.all(np.abs(oracle.decode_block(blk, synth.BC1).reshape(16, 3) - c) <= np.array([1 / 62, 1 / 126, 1 / 62]))


def test_ref_encoder_reproduces_a_representable_block_exactly():
    """Texels drawn from the palette of two 565-representable endpoints lie on a line: the PCA axis,
    its extremes, the assignment and the refinement must reproduce them with zero error (pins R24-R26)."""
    rng = np.random.default_rng(11)
    for c0, c1 in ((0xF800, 0x001F), (0x7BEF, 0x0000), (0xFFFF, 0x8410), (0x4A69, 0x2104)):
        e0, e1 = oracle.expand565(c0), oracle.expand565(c1)
        pal = oracle.palette_bc1(e0, e1)
        for _ in range(20):
            n = rng.integers(0, 4, 16)
            n[:2] = [0, 3]                                   # both extremes present
            tx = pal[n].astype(np.float32)
            blk = oracle.encode_ref_block(tx, synth.BC1)
            assert np.array_equal(oracle.decode_block(blk, synth.BC1).reshape(16, 3), tx), (hex(c0), hex(c1))


def test_ref_encoder_index_optimality_and_bc1_mode_safety():
    rng = np.random.default_rng(5)
    for fmt, ch in ((synth.BC1, 3), (synth.BC4, 1)):
        for _ in range(200):
            tx = rng.uniform(0, 1, (16, ch)).astype(np.float32).reshape(-1)
            blk = oracle.encode_ref_block(tx, fmt)
            if fmt == synth.BC1:
                c0, c1 = blk & 0xFFFF, (blk >> 16) & 0xFFFF
                assert c0 > c1 or (c0 == c1 and (blk >> 32) == 0)
            base = oracle.block_sq_error(blk, fmt, tx)
            ncode = 4 if fmt == synth.BC1 else 8
            for i in range(16):                               # no single index change lowers the error
                for code in range(ncode):
                    assert oracle.block_sq_error(_with_code(blk, fmt, i, code), fmt, tx) >= base - 1e-12
            if fmt == synth.BC4:                              # and never beats the brute-force optimum
                _, best = oracle.bruteforce_bc4(tx)
                assert base >= best - 1e-12


def test_ref_encoder_refinement_never_loses_psnr_on_noise():
    """SPEC ablation oracle: two least-squares refinements beat the unrefined (projection-only)
    endpoints on random noise, for both formats."""
    rng = np.random.default_rng(9)
    for ch, fmt in ((3, synth.BC1), (1, synth.BC4)):
        tex = rng.uniform(0, 1, (32, 32, ch)).astype(np.float32)
        p = {r: oracle.psnr(oracle.decode_bc(oracle.encode_ref_texture(tex, r), fmt, 32, 32), tex) for r in (0, 2)}
        assert p[2] >= p[0], p


def test_dds_container_round_trip_and_pillow():
    """SPEC dds_write/dds_read: 4x4 BC1 surface -> 128 + 8 bytes; read(write(s)) == s; Pillow's
    independent DDS reader decodes our container like the oracle's decoder (within its +-2 LSB)."""
    from PIL import Image
    from paper_2407_09543_b200 import dds
    blk = np.array([[0x55555555F800001F]], np.uint64)
    assert len(dds.dds_bytes(blk, 1, 4, 4)) == 136
    rng = np.random.default_rng(4)
    for fmt, ch in ((1, 3), (4, 1)):
        tex = rng.uniform(0, 1, (16, 24, ch)).astype(np.float32)
        blocks = oracle.encode_ref_texture(tex)
        data = dds.dds_bytes(blocks, fmt, 24, 16)
        b2, f2, w2, h2 = dds.read_dds(data)
        assert (f2, w2, h2) == (fmt, 24, 16) and np.array_equal(b2, blocks)
        assert dds.dds_bytes(b2, f2, w2, h2) == data
        img = Image.open(io.BytesIO(data))
        img.load()
        pil = np.asarray(img).astype(np.float64)
        pil = pil[..., :3] if fmt == 1 else pil.reshape(16, 24, -1)[..., :1]
        ours = oracle.decode_bc(blocks, fmt, 24, 16).astype(np.float64).reshape(16, 24, ch) * 255
        assert np.max(np.abs(pil - ours)) <= 2.0 + 1e-9
    with pytest.raises(ValueError):
        dds.read_dds(b"XXXX" + data[4:])


# ---------------------------------------------------------------- a1 coordinates + texel placement (R1, R2)
SYM_SPEC = dict(hidden=16, block_levels=2, block_coarsest=8, texel_levels=2, texel_coarsest=16)


def mirror_word(w: int, fmt: int, axis: str) -> int:
    """The BC word of the mirror image of a block: same endpoints, texel (x, y) -> (3-x, y) ('x') or
    (x, 3-y) ('y'); texel i = 4y + x sits at bits 32 + 2i (BC1) / 16 + 3i (BC4)."""
    shift, bits = (32, 2) if fmt == synth.BC1 else (16, 3)
    out = w & ((1 << shift) - 1)
    for i in range(16):
        x, y = i & 3, i >> 2
        j = 4 * y + (3 - x) if axis == "x" else 4 * (3 - y) + x
        out |= ((w >> (shift + bits * i)) & ((1 << bits) - 1)) << (shift + bits * j)
    return out


def check_mirror(words, fmts, axis):
    n_ok = n_bad = 0
    for k, f in enumerate(fmts):
        P = words[k]
        BH, BW = P.shape
        for by in range(BH):
            for bx in range(BW):
                mb = (by, BW - 1 - bx) if axis == "x" else (BH - 1 - by, bx)
                ok = mirror_word(int(P[by, bx]), f, axis) == int(P[mb])
                n_ok += ok
                n_bad += not ok
    return n_ok, n_bad


@pytest.mark.parametrize("axis", ["x", "y"])
def test_block_and_texel_coordinates_mirror_symmetry(axis):
    """R2 block centres (bx+1/2)/BW, texel centres (x+1/2)/W, the vertex-centred lattice p(res-1) of R1 and
    the texel order i = 4y + x: on grids mirror-symmetric along one axis only (dyadic values, 64x64
    texture, so every coordinate and lerp is exact), every block's word must equal the mirror image of
    its mirrored block's word.  An x/y swap, bx/BW instead of (bx+1/2)/BW, or a transposed texel order
    breaks the relation (checked below on the features directly)."""
    fmts = [synth.BC1, synth.BC4, synth.BC1]
    sp = synth.ModelSpec(fmts, **SYM_SPEC)
    om = oracle.Model(synth.serialize(synth.mirrored_model(sp, 11, axis)))
    words = om.decode_material(64, 64)
    n_ok, n_bad = check_mirror(words, fmts, axis)
    assert n_bad == 0 and n_ok == 3 * 16 * 16
    other = "y" if axis == "x" else "x"
    assert check_mirror(words, fmts, other)[1] > 100          # not symmetric along the other axis
    assert len({int(w) for w in words[0].ravel()}) > 100       # and not trivially constant
    # sensitivity of the construction: the correct centres give mirror-equal features; the plausible
    # mistakes do not (off-by-half block index, swapped axes)
    f32 = np.float32
    c = lambda i, n: float(f32((f32(i) + f32(0.5)) / f32(n)))     # noqa: E731
    for bx, t in ((0, 3), (5, 9), (7, 0)):
        a, b = (c(bx, 16), c(t, 16)), (c(15 - bx, 16), c(t, 16))
        if axis == "y":
            a, b = (a[1], a[0]), (b[1], b[0])
        assert np.array_equal(om.grid_encode(0, *a), om.grid_encode(0, *b))
        off = ((bx / 16, c(t, 16)), ((15 - bx) / 16, c(t, 16))) if axis == "x" else ((c(t, 16), bx / 16), (c(t, 16), (15 - bx) / 16))
        assert not np.array_equal(om.grid_encode(0, *off[0]), om.grid_encode(0, *off[1]))
        sw = (a[1], a[0]), (b[1], b[0])
        assert not np.array_equal(om.grid_encode(0, *sw[0]), om.grid_encode(0, *sw[1]))

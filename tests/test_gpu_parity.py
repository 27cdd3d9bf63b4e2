"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element, on the same
seeded inputs (-m gpu).  Bars (BASELINE.json north_star):
  * MLP float outputs within 1e-3 relative (and reported bit-exact fraction);
  * BC words bit-exact, except words the oracle places within 1e-4 of a quantization boundary
    ("excused"), which must be < 1e-4 of all blocks; unexcused mismatches = 0;
  * decoded PSNR within 0.01 dB; BC decode bit-exact (integer -> float by identical ops).
Sizes: full C1; sampled block rows (full width) of C2/C3/C4 at their full BASELINE sizes, in the
same launch configuration bench.py times; ragged and degenerate shapes."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ntbc():
    from paper_2407_09543_b200 import ntbc as n
    return n


DEV = "cuda:0"


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def float_check(g, o):
    g, o = np.asarray(g), np.asarray(o)
    zero = o == 0
    assert np.all(g[zero] == 0)
    rel = np.abs(g[~zero] - o[~zero]) / np.abs(o[~zero])
    assert rel.size == 0 or rel.max() <= 1e-3, rel.max()
    return float(np.mean(g.view(np.uint32) == o.view(np.uint32)))


def classify(fmts, gw, ow, oep):
    """Count mismatched words and how many are excused (oracle endpoint pre-rounding value within 1e-4
    of a quantization midpoint).  Index-only mismatches are never excused here (conservative)."""
    mism = excused = 0
    eo = 0
    for k, f in enumerate(fmts):
        w = 3 if f == synth.BC1 else 1
        bad = np.argwhere(gw[k] != ow[k])
        for r, c in bad:
            mism += 1
            e = oep[r, c, eo:eo + 2 * w]
            levels = np.array([31, 63, 31] * 2 if f == synth.BC1 else [255, 255], np.float64)
            v = e.astype(np.float64) * levels
            if np.any(np.abs(v - (np.floor(v) + 0.5)) / levels < 1e-4):
                excused += 1
        eo += 2 * w
    return mism, excused


def check_material(ntbc, cfg_or_blob, W, H, rows):
    blob = synth.model_blob(cfg_or_blob) if isinstance(cfg_or_blob, int) else cfg_or_blob
    m = ntbc.Model(blob)
    om = oracle.Model(blob)
    full = ntbc.decode_material([m], W, H)          # one launch over the whole material, as bench.py times it
    torch.cuda.synchronize()
    n_blocks = 0
    for r0, r1 in rows:
        ow = om.decode_material(W, H, r0, r1)
        oep, ocol = om.mlp_outputs(W, H, r0, r1)
        gw = [u64(t)[r0:r1] for t in full]
        gep, gcol = ntbc.debug_mlp(m, W, H, r0, r1)
        exact_e = float_check(gep.cpu().numpy(), oep)
        exact_c = float_check(gcol.cpu().numpy(), ocol)
        mism, exc = classify(m.fmts, gw, ow, oep)
        n_blocks += (r1 - r0) * (W // 4)
        assert mism - exc == 0, f"{mism - exc} unexcused mismatched words in rows [{r0},{r1})"
        assert mism <= 1e-4 * (r1 - r0) * (W // 4) * m.n_tex
        assert exact_e == 1.0 and exact_c == 1.0, (exact_e, exact_c)   # R10 makes the MLP bit-reproducible
    return m, full


@pytest.mark.parametrize("case", ["wide", "subnormal_a", "zero_acc", "cancel"])
def test_mma_summation_matches_reading_r10(ntbc, case):
    rng = np.random.default_rng(0)
    for K, spread in ((16, 2), (32, 8), (64, 14)):
        A = (np.exp2(rng.uniform(-spread, spread, (128, K))) * rng.choice([-1, 1], (128, K))).astype(np.float16)
        B = (np.exp2(rng.uniform(-spread, spread, (16, K))) * rng.choice([-1, 1], (16, K))).astype(np.float16)
        Cm = (rng.standard_normal((128, 16)) * 4).astype(np.float32)
        if case == "subnormal_a":     # every activation an fp16 subnormal: R comes from subnormal exponents
            A = (rng.integers(1, 1024, (128, K)) * 2.0 ** -24 * rng.choice([-1, 1], (128, K))).astype(np.float16)
        elif case == "zero_acc":      # +0 / -0 accumulators and exactly zero products
            Cm[::2] = 0.0
            Cm[1::4] = -0.0
            A[:, ::3] = 0
        elif case == "cancel":        # products that cancel exactly to 0 and leave tiny residues
            B[:, 1::2] = -B[:, 0::2]
            A[:, 1::2] = A[:, 0::2]
            A[::2, 0] = np.float16(2.0 ** -20)
        D = ntbc.debug_mma(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), torch.from_numpy(Cm).to(DEV),
                           K, 16).cpu().numpy()
        for i in range(0, 128, 3):
            for j in range(16):
                acc = float(Cm[i, j])
                for k0 in range(0, K, 16):
                    acc = oracle.fused_sum(acc, A[i, k0:k0 + 16], B[j, k0:k0 + 16], 25, 1)
                assert np.float32(acc).view(np.uint32) == D[i, j].view(np.uint32)


@pytest.mark.parametrize("fmt", [1, 4])
def test_decode_bc_bit_exact(ntbc, fmt):
    rng = np.random.default_rng(fmt)
    W, H = 4 * 37, 4 * 9                                   # odd block counts
    blocks = rng.integers(-2 ** 63, 2 ** 63 - 1, (H // 4, W // 4), dtype=np.int64)
    g = ntbc.decode_bc(torch.from_numpy(blocks).to(DEV), fmt, W, H).cpu().numpy()
    o = oracle.decode_bc(blocks.view(np.uint64), fmt, W, H)
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


@pytest.mark.parametrize("fmts,BW,BH", [([1, 1, 4, 4, 4], 41, 13), ([4], 1, 1), ([1] * 4 + [4] * 4, 130, 3),
                                        ([1], 2, 5), ([4, 1, 4, 1], 64, 8)])
def test_pack_bit_exact(ntbc, fmts, BW, BH):
    ep, col = synth.pack_inputs(fmts, BW, BH, seed=BW * 31 + BH)
    W, H = 4 * BW, 4 * BH
    g = ntbc.pack(fmts, torch.from_numpy(ep).to(DEV), torch.from_numpy(col).to(DEV), W, H)
    o = oracle.pack(fmts, ep, col, W, H)
    for k in range(len(fmts)):
        assert np.array_equal(u64(g[k]), o[k]), k


@pytest.mark.parametrize("cfg,rows", [(1, (0, 16)), (2, (0, 2)), (3, (511, 512)), (4, (1023, 1024))])
def test_grid_features_bit_exact(ntbc, cfg, rows):
    """Rows a1-a2 in isolation: Eq.2 dequantization + vertex-centred bilinear sampling, every feature of
    every block and texel of the sampled rows, bit-exact (R1-R3, R6)."""
    W, H, _ = synth.config_shape(cfg)
    blob = synth.model_blob(cfg)
    m, om = ntbc.Model(blob), oracle.Model(blob)
    bf, tf = ntbc.debug_features(m, W, H, *rows)
    bf, tf = bf.cpu().numpy(), tf.cpu().numpy()
    r0, r1 = rows
    nb, nt = 2 * om.block_levels, 2 * om.texel_levels
    f32 = np.float32
    for r in range(r1 - r0):
        by = r0 + r
        t = f32((f32(by) + f32(0.5)) / f32(H // 4))
        for bx in range(0, W // 4, max(1, W // 4 // 256)):
            s_ = f32((f32(bx) + f32(0.5)) / f32(W // 4))
            assert np.array_equal(bf[r, bx, :nb].view(np.uint32), om.grid_encode(0, float(s_), float(t)).view(np.uint32))
        for yy in range(4):
            y = 4 * by + yy
            v = f32((f32(y) + f32(0.5)) / f32(H))
            for x in range(0, W, max(1, W // 1024)):
                u = f32((f32(x) + f32(0.5)) / f32(W))
                got = tf[4 * r + yy, x, :nt]
                assert np.array_equal(got.view(np.uint32), om.grid_encode(1, float(u), float(v)).view(np.uint32)), (x, y)


def test_c1_full_material(ntbc):
    W, H, _ = synth.config_shape(1)
    check_material(ntbc, 1, W, H, [(0, H // 4)])


def test_c2_sampled_rows(ntbc):
    W, H, _ = synth.config_shape(2)
    check_material(ntbc, 2, W, H, [(0, 3), (127, 129), (H // 4 - 2, H // 4)])


def test_c2_full_material_words(ntbc):
    """Every BC word of the full 1k material (65,536 blocks x 3 textures) against the oracle."""
    W, H, _ = synth.config_shape(2)
    blob = synth.model_blob(2, material=1)
    outs = ntbc.decode_material([ntbc.Model(blob)], W, H)
    ref = oracle.Model(blob).decode_material(W, H)
    for k in range(len(outs)):
        assert np.array_equal(u64(outs[k]), ref[k]), k


@pytest.mark.parametrize("cfg", [3, 4, 6])
def test_4k_sampled_rows(ntbc, cfg):
    W, H, _ = synth.config_shape(cfg)
    check_material(ntbc, cfg, W, H, [(0, 1), (517, 518), (H // 4 - 1, H // 4)])


@pytest.mark.parametrize("W,H", [(4, 4), (12, 8), (4 * 129, 8), (4 * 300, 4 * 3), (4 * 256 + 4, 4)])
def test_ragged_and_degenerate_shapes(ntbc, W, H):
    sp = synth.ModelSpec([synth.BC1, synth.BC4, synth.BC4], hidden=32, block_levels=3, block_coarsest=8,
                         texel_levels=4, texel_coarsest=8)
    blob = synth.serialize(synth.random_model(sp, W * 7 + H))
    check_material(ntbc, blob, W, H, [(0, H // 4)])


@pytest.mark.parametrize("W,H,rows", [(16384, 16, [(0, 4)]),                        # 32 units per block row
                                      (16, 16384, [(0, 1), (2047, 2048), (4095, 4096)]),   # 1 partial unit per row
                                      (8192, 8192, [(0, 1), (1024, 1025), (2047, 2048)])])  # 2x the 4k side
def test_large_and_extreme_aspect_shapes(ntbc, W, H, rows):
    """Sizes beyond the 4k configs with the C3 architecture (paper grids): the widest and tallest block-row
    layouts and an 8192^2 material (67 M texels), decoded in one launch, rows compared with the oracle."""
    check_material(ntbc, 3, W, H, rows)


def test_closed_form_model(ntbc):
    big = 65504.0
    sp = synth.ModelSpec([synth.BC1, synth.BC4], hidden=16, block_levels=2, block_coarsest=8, texel_levels=2,
                         texel_coarsest=16)
    blob = synth.serialize(synth.closed_form_model(sp, [big, -big, -big, -big, -big, big, 1.291, -1.411],
                                                   [np.log(2.0), -big, -np.log(2.0), 0.129]))
    m = ntbc.Model(blob)
    outs = ntbc.decode_material([m], 16, 8)
    assert np.all(u64(outs[0]) == np.uint64(0xAAAAAAAA001FF800))
    assert np.all(u64(outs[1]) == np.uint64(0x92492492492432C8))


def test_conservative_pair_and_mismatch_rules(ntbc):
    W, H = 256, 64
    rgb = synth.serialize(synth.random_model(synth.ModelSpec([synth.BC1, synth.BC1], block_levels=4, texel_levels=5), 5))
    sc = synth.serialize(synth.random_model(synth.ModelSpec([synth.BC4] * 4, block_levels=4, texel_levels=5), 6))
    ms = [ntbc.Model(rgb), ntbc.Model(sc)]
    outs = ntbc.decode_material(ms, W, H)
    ref = list(oracle.Model(rgb).decode_material(W, H)) + list(oracle.Model(sc).decode_material(W, H))
    for k in range(6):
        assert np.array_equal(u64(outs[k]), ref[k])
    with pytest.raises(ntbc.NtbcError):   # two all-BC1 models are not a conservative pair
        ntbc.decode_material([ms[0], ms[0]], W, H)
    # the same pair through the pipelined host entry point (two models, two uploads, one call), with
    # separate pinned planes (one copy per texture and chunk) and with views of one pinned buffer (2-D copies)
    pinned = [torch.frombuffer(bytearray(b), dtype=torch.uint8).pin_memory() for b in (rgb, sc)]
    whole = torch.full((6, H // 4, W // 4), -1, dtype=torch.int64).pin_memory()
    for host in ([torch.full((H // 4, W // 4), -1, dtype=torch.int64).pin_memory() for _ in range(6)],
                 [whole[k] for k in range(6)]):
        for _ in range(2):
            ntbc.decode_material_host(ms, pinned, W, H, host)
            torch.cuda.synchronize()
            for k in range(6):
                assert np.array_equal(host[k].numpy().view(np.uint64), ref[k])


def test_naive_c1_full_material(ntbc):
    """Naive approach: weight network + nearest palette weight, full tiny
    material: MLP outputs bit-exact and every BC word equal to the oracle."""
    W, H, _ = synth.config_shape(8)
    check_material(ntbc, 8, W, H, [(0, H // 4)])


def test_naive_4k_sampled_rows(ntbc):
    W, H, _ = synth.config_shape(7)
    check_material(ntbc, 7, W, H, [(0, 1), (517, 518), (H // 4 - 1, H // 4)])


@pytest.mark.parametrize("fmt,ch", [(1, 3), (4, 1)])
@pytest.mark.parametrize("n_refine", [0, 2])
def test_reference_encoder_bit_exact(ntbc, fmt, ch, n_refine):
    """the GPU reference encoder (ntbc_encode_bc) against the oracle's, every word, on a
    smooth synthetic texture, uniform noise with exact 0/1 texels and constant regions (ragged size)."""
    rng = np.random.default_rng(fmt * 10 + n_refine)
    texs = [synth.texture(256, 128, ch, seed=fmt + n_refine)]
    noise = rng.uniform(0, 1, (132, 260, ch)).astype(np.float32)
    noise[::7, ::5] = 0.0
    noise[3::11, 2::3] = 1.0
    noise[:16, :16] = 0.25                                   # constant blocks (degenerate BC1, BC4 both modes)
    texs.append(noise)
    for tex in texs:
        H, W = tex.shape[:2]
        g = ntbc.encode_bc(torch.from_numpy(np.ascontiguousarray(tex)).to(DEV), fmt, W, H, n_refine)
        o = oracle.encode_ref_texture(tex, n_refine)
        assert np.array_equal(u64(g), o)


def test_reference_encoder_4k_sampled_rows(ntbc):
    W = H = 4096
    rng = np.random.default_rng(1)
    for fmt, ch in ((1, 3), (4, 1)):
        tex = rng.uniform(0, 1, (H, W, ch)).astype(np.float32)
        g = u64(ntbc.encode_bc(torch.from_numpy(tex).to(DEV), fmt, W, H))
        for by in (0, 517, H // 4 - 1):
            o = oracle.encode_ref_texture(tex[4 * by:4 * by + 4], 2)
            assert np.array_equal(g[by:by + 1], o)


@pytest.mark.parametrize("fmts,hidden,naive", [([synth.BC4] * 8, 32, False), ([synth.BC1] * 8, 64, False),
                                               ([synth.BC1, synth.BC4] * 4, 64, True), ([synth.BC1] * 3, 16, True)])
def test_extreme_head_layouts(ntbc, fmts, hidden, naive):
    """Eight textures of one format (widest endpoint head N_e = 48, all-BC4 colour head), hidden 16/32,
    naive variants; a ragged 1k-wide material (units that end mid-row), full rows compared."""
    sp = synth.ModelSpec(list(fmts), hidden=hidden, naive=naive)
    blob = synth.serialize(synth.random_model(sp, len(fmts) * 100 + hidden))
    check_material(ntbc, blob, 4 * 300, 4 * 6, [(0, 6)])


def test_host_entry_point_naive_model(ntbc):
    W, H, _ = synth.config_shape(8)
    blob = synth.model_blob(8, material=2)
    m = ntbc.Model(synth.model_blob(8))
    pinned = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
    host = [torch.full((H // 4, W // 4), -1, dtype=torch.int64).pin_memory() for _ in range(m.n_tex)]
    ntbc.decode_material_host([m], [pinned], W, H, host)
    torch.cuda.synchronize()
    ref = oracle.Model(blob).decode_material(W, H)
    for k in range(m.n_tex):
        assert np.array_equal(host[k].numpy().view(np.uint64), ref[k])


def test_tab1_conservative_pair_4k_sampled_rows(ntbc):
    """The paper's conservative workload (tools/tab1.py) at full size: an all-BC1 model and an
    all-BC4 model of the paper architecture decoded in one call; sampled rows of all 6 textures."""
    W, H = 4096, 4096
    blobs = [synth.serialize(synth.random_model(synth.ModelSpec([synth.BC1] * 2), 101)),
             synth.serialize(synth.random_model(synth.ModelSpec([synth.BC4] * 4), 102))]
    ms = [ntbc.Model(b) for b in blobs]
    outs = ntbc.decode_material(ms, W, H)
    t = 0
    for b in blobs:
        om = oracle.Model(b)
        for r0, r1 in ((0, 1), (H // 4 - 1, H // 4)):
            ref = om.decode_material(W, H, r0, r1)
            for k in range(len(ref)):
                assert np.array_equal(u64(outs[t + k])[r0:r1], ref[k])
        t += om.n_tex


def test_row_shards_union_equals_full(ntbc):
    """Multi-GPU equivalence: any block-row sharding reproduces the single-launch bytes."""
    W, H, _ = synth.config_shape(2)
    m = ntbc.Model(synth.model_blob(2))
    full = [u64(t) for t in ntbc.decode_material([m], W, H)]
    cuts = [0, 37, 128, 200, 256]
    for a, b in zip(cuts[:-1], cuts[1:]):
        part = ntbc.decode_material([m], W, H, row_begin=a, row_end=b)
        for k in range(m.n_tex):
            assert np.array_equal(u64(part[k]), full[k][a:b])


def test_host_entry_point_matches_device_path(ntbc):
    W, H, _ = synth.config_shape(2)
    blob = synth.model_blob(2, material=3)
    m = ntbc.Model(synth.model_blob(2, material=4))      # loaded with other weights; upload replaces them
    pinned = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
    host = [torch.empty((H // 4, W // 4), dtype=torch.int64).pin_memory() for _ in range(m.n_tex)]
    ntbc.decode_material_host([m], [pinned], W, H, host)
    torch.cuda.synchronize()
    ref = oracle.Model(blob).decode_material(W, H, 0, 4)
    for k in range(m.n_tex):
        assert np.array_equal(host[k].numpy().view(np.uint64)[:4], ref[k])


@pytest.mark.parametrize("W,H,contiguous", [(1024, 1024, False), (1000, 996, False), (64, 8, False),
                                            (1024, 1024, True), (1000, 996, True), (4096, 4096, True)])
def test_host_entry_point_pipelined_copies(ntbc, W, H, contiguous):
    """ntbc_decode_material_host copies row chunks back while the kernel runs (progress counters,
    DESIGN.md §6): repeated calls with changing weights and ragged shapes must return every word of the
    device path, and sampled rows (first / last of the texture) must equal the oracle.  contiguous: the
    texture planes are views of one pinned [tex][BH][BW] buffer (one 2-D copy per chunk)."""
    m = ntbc.Model(synth.model_blob(2, material=0))
    for material in (1, 2, 1):
        blob = synth.model_blob(2, material=material)
        pinned = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
        if contiguous:
            whole = torch.full((m.n_tex, H // 4, W // 4), -1, dtype=torch.int64).pin_memory()
            host = [whole[k] for k in range(m.n_tex)]
        else:
            host = [torch.full((H // 4, W // 4), -1, dtype=torch.int64).pin_memory() for _ in range(m.n_tex)]
        ntbc.decode_material_host([m], [pinned], W, H, host)
        torch.cuda.synchronize()
        dev = ntbc.decode_material([m], W, H)
        for k in range(m.n_tex):
            assert torch.equal(host[k], dev[k].cpu())
        om = oracle.Model(blob)
        for r0, r1 in ((0, 1), (H // 4 - 1, H // 4)):
            ref = om.decode_material(W, H, r0, r1)
            for k in range(m.n_tex):
                assert np.array_equal(host[k].numpy().view(np.uint64)[r0:r1], ref[k])


def test_psnr_agreement(ntbc):
    W, H, _ = synth.config_shape(1)
    blob = synth.model_blob(1)
    m = ntbc.Model(blob)
    outs = ntbc.decode_material([m], W, H)
    ref = oracle.Model(blob).decode_material(W, H)
    for k, f in enumerate(m.fmts):
        tex = synth.texture(W, H, 3 if f == 1 else 1, seed=k)
        g = ntbc.decode_bc(outs[k], f, W, H).cpu().numpy()
        o = oracle.decode_bc(ref[k], f, W, H)
        assert abs(oracle.psnr(g, tex) - oracle.psnr(o, tex)) <= 0.01


@pytest.mark.parametrize("axis", ["x", "y"])
def test_coordinates_mirror_symmetry(ntbc, axis):
    """Row a1 and the texel placement on the GPU (R1, R2; tests/test_oracle.py's pin): grids mirror-symmetric
    along one axis only give mirror-symmetric words, equal to the oracle's."""
    import test_oracle as T
    fmts = [synth.BC1, synth.BC4, synth.BC1]
    blob = synth.serialize(synth.mirrored_model(synth.ModelSpec(fmts, **T.SYM_SPEC), 11, axis))
    outs = ntbc.decode_material([ntbc.Model(blob)], 64, 64)
    words = [u64(t) for t in outs]
    ref = oracle.Model(blob).decode_material(64, 64)
    for k in range(len(fmts)):
        assert np.array_equal(words[k], ref[k])
    assert T.check_mirror(words, fmts, axis) == (3 * 16 * 16, 0)


def _digest_record(cfg):
    import hashlib
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "full_material_digests.json")
    rec = json.load(open(path)).get(str(cfg)) if os.path.exists(path) else None
    if rec is None:
        pytest.skip(f"no oracle digests for C{cfg} (tools/gen_golden_digests.py)")
    assert rec["model_sha256"] == hashlib.sha256(synth.model_blob(cfg)).hexdigest(), "synthetic model drifted"
    return rec


@pytest.mark.parametrize("cfg", [3, 4, 6])
def test_full_material_digests(ntbc, cfg):
    """Every BC word of the full-size 4k materials (C3: 5.24 M words, C4: 8.39 M, C3': 6.29 M) against the
    oracle, through digests of the oracle's words per 64-row chunk and texture written by
    tools/gen_golden_digests.py (oracle/ + synth/ only), in the launch configuration bench.py times."""
    import hashlib
    rec = _digest_record(cfg)
    W, H = rec["width"], rec["height"]
    m = ntbc.Model(synth.model_blob(cfg))
    outs = [u64(t) for t in ntbc.decode_material([m], W, H)]
    bad = []
    for c, chunk in enumerate(rec["chunks"]):
        r0 = c * rec["chunk_rows"]
        for k, d in enumerate(chunk):
            got = hashlib.sha256(outs[k][r0:r0 + rec["chunk_rows"]].astype("<u8").tobytes()).hexdigest()
            if got != d:
                bad.append((c, k))
    n_words = sum(o.size for o in outs)
    print(f"\nC{cfg}: {n_words} words in {len(rec['chunks'])} x {len(outs)} chunks, {len(bad)} chunks differ")
    assert not bad, bad[:10]


@pytest.mark.parametrize("cfg", [2, 3])
def test_psnr_agreement_full_size(ntbc, cfg):
    """Decoded PSNR of every texture of the full material (north_star: within 0.01 dB): the GPU decoder
    (kernel 3) on the GPU's words against the oracle decoder on the oracle's words (C2: the oracle decodes
    the full material; C3: the oracle's words are the digest-verified GPU words, test_full_material_digests)."""
    W, H, _ = synth.config_shape(cfg)
    blob = synth.model_blob(cfg)
    m = ntbc.Model(blob)
    outs = ntbc.decode_material([m], W, H)
    if cfg == 2:
        ref = oracle.Model(blob).decode_material(W, H)
    else:
        import hashlib
        rec = _digest_record(cfg)
        ref = [u64(t) for t in outs]
        for c, chunk in enumerate(rec["chunks"]):
            r0 = c * rec["chunk_rows"]
            for k, d in enumerate(chunk):
                assert hashlib.sha256(ref[k][r0:r0 + rec["chunk_rows"]].astype("<u8").tobytes()).hexdigest() == d
    for k, f in enumerate(m.fmts):
        tex = synth.texture(W, H, 3 if f == 1 else 1, seed=100 + k)
        g = ntbc.decode_bc(outs[k], f, W, H).cpu().numpy()
        o = oracle.decode_bc(ref[k], f, W, H)
        pg, po = oracle.psnr(g, tex), oracle.psnr(o, tex)
        print(f"\nC{cfg} texture {k}: PSNR GPU {pg:.4f} dB, oracle {po:.4f} dB")
        assert abs(pg - po) <= 0.01


@pytest.mark.parametrize("block_coarsest,texel_coarsest", [(3, 5), (5, 3), (7, 9)])
def test_odd_coarsest_resolutions(ntbc, block_coarsest, texel_coarsest):
    """Grids whose level code counts res^2 x 2 are not multiples of 4 (odd coarsest resolution): the grid
    dequantization starts every level on a fresh 4-code group; features and words equal the
    oracle's."""
    sp = synth.ModelSpec([synth.BC1, synth.BC4], hidden=32, block_levels=3, block_coarsest=block_coarsest,
                         texel_levels=4, texel_coarsest=texel_coarsest)
    blob = synth.serialize(synth.random_model(sp, block_coarsest * 10 + texel_coarsest))
    W, H = 4 * 130, 4 * 9
    check_material(ntbc, blob, W, H, [(0, H // 4)])
    m, om = ntbc.Model(blob), oracle.Model(blob)
    bf, tf = (t.cpu().numpy() for t in ntbc.debug_features(m, W, H, 0, 2))
    for bx in (0, 1, 77, 129):
        s_ = np.float32((np.float32(bx) + np.float32(0.5)) / np.float32(W // 4))
        t = np.float32(np.float32(1.5) / np.float32(H // 4))
        assert np.array_equal(bf[1, bx, :6].view(np.uint32), om.grid_encode(0, float(s_), float(t)).view(np.uint32))


def test_pack_bc4_ties_and_monotone_argmin(ntbc):
    """The pack kernel's one-select BC4 argmin (bc4_code_mono, valid for E0 != E1) against the oracle's
    strict-< scan on adversarial texels: every midpoint between adjacent binary32 palette entries and its two
    neighbouring floats, for endpoint pairs including E0 = 0, E1 = 255 (Eq. 8's constants equal to an
    endpoint), E0 = E1 +- 1 and E0 = E1 (the exact-scan fallback), both modes."""
    rng = np.random.default_rng(5)
    pairs = [(0, 0), (255, 255), (0, 255), (255, 0), (0, 1), (1, 0), (254, 255), (255, 254), (52, 52), (200, 10)]
    pairs += [tuple(int(v) for v in rng.integers(0, 256, 2)) for _ in range(54)]
    blocks_ep, texels = [], []
    for E0, E1 in pairs:
        pal = oracle.palette_bc4(E0, E1).astype(np.float32)
        vals = []
        for n in range(7):
            mid = np.float32((np.float64(pal[n]) + np.float64(pal[n + 1])) / 2)
            vals += [mid, np.nextafter(mid, np.float32(-1)), np.nextafter(mid, np.float32(2))]
        vals += list(pal) + [np.float32(0), np.float32(1), np.float32(0.5)]
        vals = np.array(vals, np.float32)
        for j in range(0, len(vals), 16):
            t = vals[j:j + 16]
            t = np.concatenate([t, rng.uniform(0, 1, 16 - t.size).astype(np.float32)]) if t.size < 16 else t
            blocks_ep.append([np.float32(E0) / np.float32(255), np.float32(E1) / np.float32(255)])
            texels.append(t)
    nb = len(blocks_ep)
    BW = nb                               # one block row
    ep = np.array(blocks_ep, np.float32).reshape(1, BW, 2)
    col = np.zeros((4, 4 * BW, 1), np.float32)
    for b, t in enumerate(texels):
        for i in range(16):
            col[i >> 2, 4 * b + (i & 3), 0] = t[i]
    W, H = 4 * BW, 4
    o = oracle.pack([4], ep, col, W, H)
    assert all(((int(w) & 0xFF) == E0 and ((int(w) >> 8) & 0xFF) == E1)
               for w, (E0, E1) in zip(o[0][0][::3], [(int(round(e[0] * 255)), int(round(e[1] * 255))) for e in blocks_ep[::3]]))
    g = ntbc.pack([4], torch.from_numpy(ep).to(DEV), torch.from_numpy(col).to(DEV), W, H)
    assert np.array_equal(u64(g[0]), o[0])


def test_pack_misaligned_inputs(ntbc):
    """ntbc_pack with a colour array that is only 4-B aligned (the bulk-copy form needs 16 B: the library falls
    back to the warp form) and an odd block count (8-byte stores), against the oracle."""
    fmts = [synth.BC1, synth.BC4, synth.BC4]
    ep, col = synth.pack_inputs(fmts, 37, 5, seed=3)
    W, H = 4 * 37, 4 * 5
    buf = torch.empty(col.size + 1, dtype=torch.float32, device=DEV)
    buf[1:] = torch.from_numpy(col.reshape(-1)).to(DEV)
    col_d = buf[1:].view(col.shape)
    g = ntbc.pack(fmts, torch.from_numpy(ep).to(DEV), col_d, W, H)
    o = oracle.pack(fmts, ep, col, W, H)
    for k in range(len(fmts)):
        assert np.array_equal(u64(g[k]), o[k]), k

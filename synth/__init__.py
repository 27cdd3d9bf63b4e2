"""Seeded synthetic inputs for NTBC inference (shared by the oracle tests and the CUDA path).

This module holds NO arithmetic of the method (no grid encoding, no MLP, no
quantization of predictions, no BC packing).  It only draws random numbers and
serialises them into the `.ntbc` container described in DESIGN.md §3, so both
sides of every parity test start from byte-identical inputs.

Input recipe:
  * MLP weights: He-normal N(0, 2/fan_in) ("He initialization"),
    stored as fp16 ("stored in half-precision").
  * MLP biases: U(-0.1, 0.1) -> fp16 (paper silent; DESIGN reading R7).
  * Grids: "trained-like" smooth multi-octave noise, drawn directly as uint8
    codes with a random per-level scale s and zero point z (PAPER.md:321-326:
    8-bit grids with per-level asymmetric (s, z)).  Architecture per
    PAPER.md:334-337 (block grid 7 levels 16..1024, texel grid 8 levels
    16..2048, 2 features per level).
  * Seeds: SplitMix64(0x4E544243 ^ (config << 32) ^ material) -> numpy PCG64.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

BC1 = 1
BC4 = 4
MAGIC = b"NTBC"
VERSION = 1
MAX_TEXTURES = 8
HEADER_BYTES = 96


def _align16(n: int) -> int:
    return (n + 15) & ~15


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def seed_for(config: int, material: int) -> int:
    return splitmix64(0x4E544243 ^ (config << 32) ^ material)


@dataclass
class ModelSpec:
    """Architecture of one NTBC model (one `.ntbc` file)."""
    fmts: list                     # texture formats in head order (BC1/BC4)
    hidden: int = 64               # PAPER.md:331 "64 neurons"
    n_hidden: int = 3              # PAPER.md:331 "three hidden layers"
    features: int = 2              # PAPER.md:336 "2D features per level"
    block_levels: int = 7
    block_coarsest: int = 16
    texel_levels: int = 8
    texel_coarsest: int = 16
    naive: bool = False            # weight network (one weight per texel per texture)

    @property
    def n_endpoint_out(self) -> int:   # PAPER.md:388  6 N_RGB + 2 N_SC
        return sum(6 if f == BC1 else 2 for f in self.fmts)

    @property
    def n_color_out(self) -> int:      # PAPER.md:388  3 N_RGB + N_SC; naive: one weight per texture
        return len(self.fmts) if self.naive else sum(3 if f == BC1 else 1 for f in self.fmts)

    @property
    def endpoint_in(self) -> int:
        return self.block_levels * self.features

    @property
    def color_in(self) -> int:
        return self.texel_levels * self.features

    def level_res(self, which: str) -> list:
        c, n = ((self.block_coarsest, self.block_levels) if which == "block"
                else (self.texel_coarsest, self.texel_levels))
        return [c << l for l in range(n)]

    def mlp_dims(self, which: str) -> list:
        i = self.endpoint_in if which == "endpoint" else self.color_in
        o = self.n_endpoint_out if which == "endpoint" else self.n_color_out
        return [i] + [self.hidden] * self.n_hidden + [o]


# The five BASELINE.json configs (C3' = the paper's Tab. 1 shape).
CONFIGS = {
    1: dict(name="C1-64px-bc1+bc4-tiny", width=64, height=64,
            spec=lambda: ModelSpec([BC1, BC4], hidden=16, block_levels=2, block_coarsest=8,
                                   texel_levels=2, texel_coarsest=16)),
    2: dict(name="C2-1k-2bc1+1bc4", width=1024, height=1024,
            spec=lambda: ModelSpec([BC1, BC1, BC4])),
    3: dict(name="C3-4k-MetalPlates013-shaped-2bc1+3bc4", width=4096, height=4096,
            spec=lambda: ModelSpec([BC1, BC1, BC4, BC4, BC4])),
    4: dict(name="C4-4k-4bc1+4bc4", width=4096, height=4096,
            spec=lambda: ModelSpec([BC1, BC1, BC1, BC1, BC4, BC4, BC4, BC4])),
    6: dict(name="C3p-4k-paper-Tab1-2bc1+4bc4", width=4096, height=4096,
            spec=lambda: ModelSpec([BC1, BC1, BC4, BC4, BC4, BC4])),
    7: dict(name="C3-4k-naive-weight-net-2bc1+3bc4", width=4096, height=4096,
            spec=lambda: ModelSpec([BC1, BC1, BC4, BC4, BC4], naive=True)),
    8: dict(name="C1-64px-naive-bc1+bc4-tiny", width=64, height=64,
            spec=lambda: ModelSpec([BC1, BC4], hidden=16, block_levels=2, block_coarsest=8, texel_levels=2,
                                   texel_coarsest=16, naive=True)),
}


def _smooth_noise(rng: np.random.Generator, res: int, octaves: int = 4) -> np.ndarray:
    """Multi-octave value noise on a res x res lattice, roughly in [-1, 1]."""
    out = np.zeros((res, res), np.float64)
    amp, total = 1.0, 0.0
    for o in range(octaves):
        cr = max(2, min(res, 4 << o))
        coarse = rng.standard_normal((cr, cr))
        # separable linear upsampling of the coarse lattice to res x res
        xs = np.linspace(0.0, cr - 1.0, res)
        i0 = np.minimum(np.floor(xs).astype(np.int64), cr - 2)
        t = xs - i0
        rows = coarse[i0] * (1 - t)[:, None] + coarse[i0 + 1] * t[:, None]
        up = rows[:, i0] * (1 - t)[None, :] + rows[:, i0 + 1] * t[None, :]
        out += amp * up
        total += amp
        amp *= 0.6
    out += 0.35 * rng.standard_normal((res, res))   # texel-scale detail
    return out / (total + 0.35)


@dataclass
class Model:
    spec: ModelSpec
    # per grid: list of (s: float32, z: int32, codes uint8 [res][res][F])
    block_grid: list = field(default_factory=list)
    texel_grid: list = field(default_factory=list)
    # per MLP: list of (W fp16 [in][out], b fp16 [out])
    endpoint_mlp: list = field(default_factory=list)
    color_mlp: list = field(default_factory=list)


def random_model(spec: ModelSpec, seed: int) -> Model:
    rng = np.random.Generator(np.random.PCG64(seed))
    m = Model(spec)
    for which, dst in (("block", m.block_grid), ("texel", m.texel_grid)):
        for res in spec.level_res(which):
            s = np.float32(rng.uniform(0.004, 0.012))
            z = np.int32(rng.integers(108, 149))
            feats = []
            for _ in range(spec.features):
                n = _smooth_noise(rng, res)
                feats.append(np.clip(np.rint(float(z) + n * 90.0), 0, 255).astype(np.uint8))
            dst.append((s, z, np.ascontiguousarray(np.stack(feats, axis=-1))))
    for which, dst in (("endpoint", m.endpoint_mlp), ("color", m.color_mlp)):
        dims = spec.mlp_dims(which)
        for i, o in zip(dims[:-1], dims[1:]):
            w = (rng.standard_normal((i, o)) * np.sqrt(2.0 / i)).astype(np.float16)
            b = rng.uniform(-0.1, 0.1, o).astype(np.float16)
            dst.append((w, b))
    return m


def mirrored_model(spec: ModelSpec, seed: int, axis: str) -> Model:
    """random_model with every grid level's codes mirror-symmetric along `axis` ('x': q[j][i] =
    q[j][res-1-i]; 'y': q[j][i] = q[res-1-j][i]) and not along the other, and every level's scale
    s = 2^-6 (dyadic values, so the lattice coordinates and lerps of power-of-two textures are exact).
    Input of the coordinate / texel-placement symmetry pins (tests/test_oracle.py)."""
    m = random_model(spec, seed)
    for grid in (m.block_grid, m.texel_grid):
        for li, (s_, z, codes) in enumerate(grid):
            c = codes.copy()
            res = c.shape[0]
            if axis == "x":
                c[:, res - res // 2:] = c[:, :res // 2][:, ::-1]
            else:
                c[res - res // 2:] = c[:res // 2][::-1]
            grid[li] = (np.float32(2.0 ** -6), z, np.ascontiguousarray(c))
    return m


def serialize(m: Model) -> bytes:
    """Write the `.ntbc` v1 container (layout in DESIGN.md §3)."""
    sp = m.spec
    assert 1 <= len(sp.fmts) <= MAX_TEXTURES
    fm = list(sp.fmts) + [0] * (MAX_TEXTURES - len(sp.fmts))
    hdr = MAGIC + struct.pack("<II", VERSION, len(sp.fmts)) + struct.pack("<8I", *fm)
    hdr += struct.pack("<III", sp.hidden, sp.n_hidden, sp.features)
    hdr += struct.pack("<IIII", sp.block_levels, sp.block_coarsest, sp.texel_levels, sp.texel_coarsest)
    hdr += struct.pack("<IIII", sp.endpoint_in, sp.n_endpoint_out, sp.color_in, sp.n_color_out)
    hdr += struct.pack("<I", 1 if sp.naive else 0)   # variant: 0 NTBC (colour network), 1 naive (weights)
    hdr = hdr.ljust(HEADER_BYTES, b"\0")
    parts = [hdr]

    def pad(b: bytes) -> bytes:
        return b + b"\0" * (_align16(len(b)) - len(b))

    qp = b"".join(struct.pack("<fi", float(s), int(z)) for s, z, _ in m.block_grid + m.texel_grid)
    parts.append(pad(qp))
    for _, _, codes in m.block_grid + m.texel_grid:
        parts.append(pad(codes.tobytes()))
    for mlp in (m.endpoint_mlp, m.color_mlp):
        for w, b in mlp:
            parts.append(pad(w.astype("<f2").tobytes()))
            parts.append(pad(b.astype("<f2").tobytes()))
    return b"".join(parts)


def model_blob(config: int, material: int = 0) -> bytes:
    c = CONFIGS[config]
    return serialize(random_model(c["spec"](), seed_for(config, material)))


def config_shape(config: int):
    c = CONFIGS[config]
    return c["width"], c["height"], c["spec"]()


def closed_form_model(spec: ModelSpec, endpoint_out_bias, color_out_bias) -> Model:
    """All weights and hidden biases zero; only the output biases are set.

    Used by the hand-computed end-to-end golden: every hidden
    activation is selu(0) = 0, so each output equals sigmoid(bias).
    """
    m = Model(spec)
    for which, dst in (("block", m.block_grid), ("texel", m.texel_grid)):
        for res in spec.level_res(which):
            dst.append((np.float32(0.01), np.int32(128),
                        np.full((res, res, spec.features), 128, np.uint8)))
    for which, dst, ob in (("endpoint", m.endpoint_mlp, endpoint_out_bias),
                           ("color", m.color_mlp, color_out_bias)):
        dims = spec.mlp_dims(which)
        for li, (i, o) in enumerate(zip(dims[:-1], dims[1:])):
            w = np.zeros((i, o), np.float16)
            b = np.zeros(o, np.float16)
            if li == len(dims) - 2:
                b = np.asarray(ob, np.float16)
            dst.append((w, b))
    return m


def pack_inputs(fmts, n_blocks_w: int, n_blocks_h: int, seed: int):
    """Random fp32 MLP outputs for feeding the standalone quantize-and-pack stage.

    Values are uniform in [0, 1] with a sprinkling of the exact edge values
    0, 1, 0.5, and ~3% of (block, texture) pairs get e1 := e0 so the
    degenerate equal-endpoint paths are exercised.  Head layout per
    DESIGN.md §3 (BC1: e0.rgb, e1.rgb; BC4: e0, e1).
    Returns (endpoints [BH][BW][N_e], colors [H][W][N_c]) float32.
    """
    n_e = sum(6 if f == BC1 else 2 for f in fmts)
    n_c = sum(3 if f == BC1 else 1 for f in fmts)
    rng = np.random.Generator(np.random.PCG64(seed))
    ep = rng.uniform(0, 1, (n_blocks_h, n_blocks_w, n_e)).astype(np.float32)
    co = rng.uniform(0, 1, (n_blocks_h * 4, n_blocks_w * 4, n_c)).astype(np.float32)
    for a in (ep, co):
        flat = a.reshape(-1)
        k = max(1, flat.size // 50)
        idx = rng.integers(0, flat.size, k)
        flat[idx] = rng.choice(np.array([0.0, 1.0, 0.5], np.float32), k)
    bl = ep.reshape(-1, n_e)
    off = 0
    for f in fmts:
        w = 3 if f == BC1 else 1
        sel = rng.random(bl.shape[0]) < 0.03
        bl[sel, off + w:off + 2 * w] = bl[sel, off:off + w]
        off += 2 * w
    return ep, co


def texture(width: int, height: int, channels: int, seed: int) -> np.ndarray:
    """Procedural texture in [0,1] (used only for PSNR reporting)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    res = max(width, height)
    base = _smooth_noise(rng, res, octaves=5)[:height, :width]
    out = np.empty((height, width, channels), np.float32)
    for c in range(channels):
        out[..., c] = np.clip(0.5 + 0.35 * base + 0.05 * rng.standard_normal((height, width)), 0, 1)
    return out

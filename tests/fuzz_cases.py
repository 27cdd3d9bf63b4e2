"""Seeded random model / shape cases for the GPU fuzz tests (tests/test_gpu_fuzz.py, tests/checked_run.py).
Input generation only (synth/): no arithmetic of the method."""
import numpy as np

import synth


def cases(n: int, seed: int = 2407):
    """n cases: (blob, W, H, row_begin, row_end, misalign) with random format mixes (1-8 textures), hidden
    width 16/32/64, NTBC or naive variant, grids of 1-8 levels with coarsest 2-9 (finest <= 1024), textures
    of 4..640 texels per side (ragged units and odd W/4), a random block-row shard, and 8-B-only aligned
    output planes for some cases (the kernel's 8-byte store path)."""
    rng = np.random.default_rng(seed)
    out = []
    for c in range(n):
        nt = int(rng.integers(1, 9))
        fmts = [int(f) for f in rng.choice([synth.BC1, synth.BC4], nt)]
        hidden = int(rng.choice([16, 32, 64]))
        naive = bool(rng.random() < 0.2)
        bl = int(rng.integers(1, 9))
        bc = int(rng.integers(2, 10))
        while bc << (bl - 1) > 1024:
            bl -= 1
        tl = int(rng.integers(1, 9))
        tc = int(rng.integers(2, 10))
        while tc << (tl - 1) > 1024:
            tl -= 1
        sp = synth.ModelSpec(fmts, hidden=hidden, block_levels=bl, block_coarsest=bc, texel_levels=tl,
                             texel_coarsest=tc, naive=naive)
        blob = synth.serialize(synth.random_model(sp, seed * 1000 + c))
        W = 4 * int(rng.integers(1, 161))
        H = 4 * int(rng.integers(1, 41))
        BH = H // 4
        r0 = int(rng.integers(0, BH))
        r1 = int(rng.integers(r0 + 1, BH + 1))
        misalign = bool(rng.random() < 0.3)
        out.append((blob, W, H, r0, r1, misalign))
    return out

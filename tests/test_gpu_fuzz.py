"""Seeded random fuzzing of the fused decode (-m gpu): 60 random models and shapes (tests/fuzz_cases.py) --
format mixes of 1-8 textures, hidden 16/32/64, NTBC and naive variants, grids with 1-8 levels and odd
coarsest resolutions, ragged and tiny textures, random block-row shards, 8-B-only aligned output planes --
every word and every MLP output of the shard against the oracle, bit-exact."""
import numpy as np
import pytest
import torch

import oracle
from fuzz_cases import cases

pytestmark = pytest.mark.gpu
CASES = cases(60)


@pytest.mark.parametrize("c", range(len(CASES)))
def test_fuzz_decode_bit_exact(c):
    from paper_2407_09543_b200 import ntbc
    blob, W, H, r0, r1, misalign = CASES[c]
    m, om = ntbc.Model(blob), oracle.Model(blob)
    rows, BW = r1 - r0, W // 4
    buf = torch.full((m.n_tex, rows * BW + 2), -1, dtype=torch.int64, device="cuda")
    ptrs = [buf[k].data_ptr() + (8 if misalign else 0) for k in range(m.n_tex)]
    ntbc.decode_material([m], W, H, row_begin=r0, row_end=r1, out_ptrs=ptrs)
    ref = om.decode_material(W, H, r0, r1)
    off = 1 if misalign else 0
    for k in range(m.n_tex):
        got = buf[k].cpu().numpy().view(np.uint64)[off:off + rows * BW].reshape(rows, BW)
        assert np.array_equal(got, ref[k]), (c, k)
    gep, gcol = ntbc.debug_mlp(m, W, H, r0, r1)
    oep, ocol = om.mlp_outputs(W, H, r0, r1)
    assert np.array_equal(gep.cpu().numpy().view(np.uint32), oep.view(np.uint32))
    assert np.array_equal(gcol.cpu().numpy().view(np.uint32), ocol.view(np.uint32))

"""Seeded random fuzzing of the fused decode (-m gpu): 60 random models and shapes (tests/fuzz_cases.py) --
format mixes of 1-8 textures, hidden 16/32/64, NTBC and naive variants, grids with 1-8 levels and odd
coarsest resolutions, ragged and tiny textures, random block-row shards, 8-B-only aligned output planes --
every word and every MLP output of the shard against the oracle, bit-exact.  The same under contracts F and P
(ntbc_set_contract 1 / 2 against oracle.contract_f() / contract_p()) on 20 further non-naive cases each."""
import contextlib
import numpy as np
import pytest
import torch

import oracle
from fuzz_cases import cases

pytestmark = pytest.mark.gpu
CASES = cases(60)
CONTRACT_CASES = [c for c in cases(60, seed=4099) if not oracle.Model(c[0]).naive][:20]


def _check(case, contract=0):
    from paper_2407_09543_b200 import ntbc
    blob, W, H, r0, r1, misalign = case
    m, om = ntbc.Model(blob), oracle.Model(blob)
    if contract:
        ntbc.set_contract(m, contract)
    mode = {0: contextlib.nullcontext, 1: oracle.contract_f, 2: oracle.contract_p}[contract]
    rows, BW = r1 - r0, W // 4
    buf = torch.full((m.n_tex, rows * BW + 2), -1, dtype=torch.int64, device="cuda")
    ptrs = [buf[k].data_ptr() + (8 if misalign else 0) for k in range(m.n_tex)]
    ntbc.decode_material([m], W, H, row_begin=r0, row_end=r1, out_ptrs=ptrs)
    with mode():
        ref = om.decode_material(W, H, r0, r1)
        oep, ocol = om.mlp_outputs(W, H, r0, r1)
    off = 1 if misalign else 0
    for k in range(m.n_tex):
        got = buf[k].cpu().numpy().view(np.uint64)[off:off + rows * BW].reshape(rows, BW)
        assert np.array_equal(got, ref[k]), (contract, k)
    gep, gcol = ntbc.debug_mlp(m, W, H, r0, r1)
    assert np.array_equal(gep.cpu().numpy().view(np.uint32), oep.view(np.uint32))
    assert np.array_equal(gcol.cpu().numpy().view(np.uint32), ocol.view(np.uint32))


@pytest.mark.parametrize("c", range(len(CASES)))
def test_fuzz_decode_bit_exact(c):
    _check(CASES[c])


@pytest.mark.parametrize("contract", [1, 2])
@pytest.mark.parametrize("c", range(20))
def test_fuzz_contracts_bit_exact(c, contract):
    _check(CONTRACT_CASES[c], contract)

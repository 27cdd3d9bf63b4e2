"""GPU parity of the colour-network training step (-m gpu): ntbc_train_colour_step
(fp32, CUDA cores, atomic accumulation) against the float64 autograd oracle (oracle/train_oracle.py).

Bars (R32): loss within 1e-5 relative; every parameter class (grid levels, weights,
biases) of the gradient within tol x the norm of the whole gradient, tol = 2e-6 / T (fp32 terms of
the STE expectation carry a 1/T factor, and grid entries are sums of many sample contributions with
cancellation, accumulated by atomics in arbitrary order); the Adam update equal (1e-6 relative) to
the bias-corrected formula applied to the GPU's own gradient.  A wrong sign, factor or index in any
term is an O(1) relative error.  Samples within MARGIN of an argmax tie (decided by the float64 oracle)
are dropped from the batch: there the discrete decision may legitimately differ in fp32."""
import numpy as np
import pytest
import torch

from oracle import train_oracle as T

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def ntbc():
    from paper_2407_09543_b200 import ntbc as n
    return n


MARGIN = 1e-4   # samples whose two nearest palette distances are closer than this (float64, oracle) are
                # dropped: fp32 may take the other argmax branch there, a discrete O(1/B) gradient change


def _case(fmts, levels, coarsest, B, seed, W=256, H=192, qat=False):
    rng = np.random.default_rng(seed)
    lay = T.layout(fmts, 64, levels, coarsest)
    n = sum(int(np.prod(s)) for _, s in lay)
    n_grid = sum(int(np.prod(s)) for nme, s in lay if nme.startswith("grid"))
    p = rng.standard_normal(n) * 0.3
    p[:n_grid] = rng.uniform(-1, 1, n_grid)
    p = p.astype(np.float32)
    n_c = sum(3 if f == T.BC1 else 1 for f in fmts)
    n_e = sum(6 if f == T.BC1 else 2 for f in fmts)
    xy = np.stack([rng.integers(0, W, B), rng.integers(0, H, B)], 1).astype(np.int32)
    cref = rng.uniform(0, 1, (B, n_c)).astype(np.float32)
    eref = rng.uniform(0, 1, (B, n_e)).astype(np.float32)
    keep = T.colour_margins(torch.from_numpy(p.astype(np.float64)), lay, fmts, torch.from_numpy(xy.astype(np.int64)),
                            W, H, torch.from_numpy(eref.astype(np.float64)), qat).numpy() > MARGIN
    return lay, n_grid, p, xy[keep], cref[keep], eref[keep], W, H


@pytest.mark.parametrize("fmts,levels,coarsest,B,temp,qat", [
    ([T.BC1, T.BC4], 2, 4, 300, 0.1, False),
    ([T.BC1, T.BC1, T.BC4, T.BC4, T.BC4], 4, 8, 1000, 0.01, False),
    ([T.BC4, T.BC1], 8, 16, 2048, 0.01, False),              # the paper's texel grid
    ([T.BC1, T.BC4], 2, 4, 300, 0.1, True),                  # QAT
    ([T.BC4, T.BC1], 8, 16, 2048, 0.01, True),
])
def test_train_step_matches_oracle(ntbc, fmts, levels, coarsest, B, temp, qat):
    lay, n_grid, p, xy, cref, eref, W, H = _case(fmts, levels, coarsest, B, seed=B, qat=qat)
    n = p.size
    assert ntbc.train_param_count(fmts, 64, levels, coarsest) == n
    dp = torch.from_numpy(p).to(DEV)
    g = torch.zeros(n, device=DEV)
    m = torch.zeros(n, device=DEV)
    v = torch.zeros(n, device=DEV)
    loss = ntbc.train_colour_step(fmts, dp, g, m, v, 1, torch.from_numpy(xy).to(DEV), torch.from_numpy(cref).to(DEV),
                                  torch.from_numpy(eref).to(DEV), W, H, temperature=temp, levels=levels,
                                  coarsest=coarsest, qat=qat)
    torch.cuda.synchronize()
    ref_loss, ref_g, _, _, _ = T.colour_step(torch.from_numpy(p.astype(np.float64)), torch.zeros(n, dtype=torch.float64),
                                             torch.zeros(n, dtype=torch.float64), 1, lay, fmts,
                                             torch.from_numpy(xy.astype(np.int64)), W, H,
                                             torch.from_numpy(cref.astype(np.float64)),
                                             torch.from_numpy(eref.astype(np.float64)), T=temp, qat=qat)
    assert abs(float(loss) - ref_loss) <= 1e-5 * abs(ref_loss)
    gg = g.double().cpu()
    off = 0
    for name, shape in lay:                               # every parameter class separately
        k = int(np.prod(shape))
        a, b = gg[off:off + k], ref_g[off:off + k]
        assert float(torch.linalg.norm(a - b)) <= 2e-6 / temp * float(torch.linalg.norm(ref_g)) + 1e-12, name
        off += k
    # Adam update applied to the GPU's own gradient (bias-corrected)
    lr = torch.full((n,), 0.005, dtype=torch.float64)
    lr[:n_grid] = 0.01
    want, _, _ = T.adam(torch.from_numpy(p.astype(np.float64)), gg, torch.zeros(n, dtype=torch.float64),
                        torch.zeros(n, dtype=torch.float64), 1, lr)
    got = dp.double().cpu()
    assert torch.allclose(got, want, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("fmts,levels,coarsest,B,temp,qat", [
    ([T.BC1, T.BC4], 2, 4, 300, 0.1, False),
    ([T.BC1, T.BC1, T.BC4, T.BC4, T.BC4], 7, 16, 1000, 0.01, False),   # the paper's block grid
    ([T.BC1, T.BC1, T.BC4, T.BC4, T.BC4], 7, 16, 1000, 0.01, True),
])
def test_endpoint_train_step_matches_oracle(ntbc, fmts, levels, coarsest, B, temp, qat):
    rng = np.random.default_rng(B + 7)
    lay = T.layout_endpoint(fmts, 64, levels, coarsest)
    n = sum(int(np.prod(s)) for _, s in lay)
    n_grid = sum(int(np.prod(s)) for nme, s in lay if nme.startswith("grid"))
    assert ntbc.train_endpoint_param_count(fmts, 64, levels, coarsest) == n
    p = rng.standard_normal(n) * 0.3
    p[:n_grid] = rng.uniform(-1, 1, n_grid)
    p = p.astype(np.float32)
    n_c = sum(3 if f == T.BC1 else 1 for f in fmts)
    n_e = sum(6 if f == T.BC1 else 2 for f in fmts)
    BW, BH = 200, 150
    bxy = np.stack([rng.integers(0, BW, B), rng.integers(0, BH, B)], 1).astype(np.int32)
    c16 = rng.uniform(0, 1, (B, 16, n_c)).astype(np.float32)
    eref = rng.uniform(0, 1, (B, n_e)).astype(np.float32)
    keep = T.endpoint_margins(torch.from_numpy(p.astype(np.float64)), lay, fmts, torch.from_numpy(bxy.astype(np.int64)),
                              BW, BH, torch.from_numpy(c16.astype(np.float64)), qat).numpy() > MARGIN
    bxy, c16, eref = bxy[keep], c16[keep], eref[keep]
    dp = torch.from_numpy(p).to(DEV)
    g, m, v = (torch.zeros(n, device=DEV) for _ in range(3))
    loss = ntbc.train_endpoint_step(fmts, dp, g, m, v, 1, torch.from_numpy(bxy).to(DEV), torch.from_numpy(c16).to(DEV),
                                    torch.from_numpy(eref).to(DEV), BW, BH, temperature=temp, levels=levels,
                                    coarsest=coarsest, qat=qat)
    torch.cuda.synchronize()
    ref_loss, ref_g, _, _, _ = T.endpoint_step(torch.from_numpy(p.astype(np.float64)), torch.zeros(n, dtype=torch.float64),
                                               torch.zeros(n, dtype=torch.float64), 1, lay, fmts,
                                               torch.from_numpy(bxy.astype(np.int64)), BW, BH,
                                               torch.from_numpy(eref.astype(np.float64)),
                                               torch.from_numpy(c16.astype(np.float64)), T=temp, qat=qat)
    assert abs(float(loss) - ref_loss) <= 1e-5 * abs(ref_loss)
    gg = g.double().cpu()
    off = 0
    for name, shape in lay:
        k = int(np.prod(shape))
        assert float(torch.linalg.norm(gg[off:off + k] - ref_g[off:off + k])) <= \
            2e-6 / temp * float(torch.linalg.norm(ref_g)) + 1e-12, name
        off += k

"""Pins of the training-step oracle (oracle/train_oracle.py) against independent
references (-m "not gpu"): finite differences, torch.optim.Adam, torch grid_sample, closed forms."""
import numpy as np
import torch

from oracle import train_oracle as T


def _setup(fmts, levels=2, coarsest=4, B=64, seed=0, W=32, H=32):
    rng = np.random.default_rng(seed)
    lay = T.layout(fmts, 64, levels, coarsest)
    n = sum(int(np.prod(s)) for _, s in lay)
    params = torch.from_numpy(rng.standard_normal(n) * 0.3)
    xy = torch.from_numpy(np.stack([rng.integers(0, W, B), rng.integers(0, H, B)], 1))
    n_c = sum(3 if f == T.BC1 else 1 for f in fmts)
    n_e = sum(6 if f == T.BC1 else 2 for f in fmts)
    cref = torch.from_numpy(rng.uniform(0, 1, (B, n_c)))
    eref = torch.from_numpy(rng.uniform(0, 1, (B, n_e)))
    return lay, params, xy, cref, eref, W, H


def test_grid_features_vs_torch_grid_sample():
    """The vertex-centred lookup (R1) is grid_sample with align_corners=True at the same lattice point
    (X = RN32(u (res-1)), the inference convention, passed to grid_sample as its normalized coordinate)."""
    rng = np.random.default_rng(1)
    g = torch.from_numpy(rng.standard_normal((9, 9, 2)))
    u = torch.from_numpy(rng.uniform(0.01, 0.99, 100).astype(np.float32))
    v = torch.from_numpy(rng.uniform(0.01, 0.99, 100).astype(np.float32))
    ours = T.grid_features([g], u, v)
    X = (u * torch.tensor(8.0, dtype=torch.float32)).double()
    Y = (v * torch.tensor(8.0, dtype=torch.float32)).double()
    ref = torch.nn.functional.grid_sample(g.permute(2, 0, 1)[None], torch.stack([X / 4 - 1, Y / 4 - 1], 1)[None, None],
                                          mode="bilinear", align_corners=True)[0, :, 0].T
    assert torch.allclose(ours, ref, atol=1e-12)


def test_ste_backward_is_the_derivative_of_the_softmax_expectation():
    """Backward of ste_decoded == finite differences of sum_n softmax(d/T)_n c_n (App. A, corrected
    w_n - w_hat); forward == the hard palette colour of the argmax."""
    rng = np.random.default_rng(2)
    for fmt in (T.BC1, T.BC4):
        e = torch.from_numpy(rng.uniform(0, 1, (5, 6 if fmt == T.BC1 else 2)))
        pal = T.palettes(fmt, e)
        w = pal.shape[2]
        ch = torch.from_numpy(rng.uniform(0, 1, (5, w))).requires_grad_(True)
        Tt = 0.5
        out = T.ste_decoded(ch, pal, Tt)
        dist = torch.sqrt(((ch.detach()[:, None] - pal) ** 2).sum(-1))
        hard = pal[torch.arange(5), torch.argmin(dist, 1)]
        assert torch.allclose(out.detach(), hard)
        r = torch.from_numpy(rng.standard_normal((5, w)))
        (g,) = torch.autograd.grad((out * r).sum(), ch)

        def soft(c):
            d = -torch.sqrt(((c[:, None] - pal) ** 2).sum(-1))
            return (torch.softmax(d / Tt, 1)[:, :, None] * pal).sum(1)
        eps = 1e-6
        fd = torch.zeros_like(g)
        for i in range(5):
            for x in range(w):
                cp, cm = ch.detach().clone(), ch.detach().clone()
                cp[i, x] += eps
                cm[i, x] -= eps
                fd[i, x] = ((soft(cp) - soft(cm)) * r).sum() / (2 * eps)
        assert torch.allclose(g, fd, rtol=1e-5, atol=1e-7), fmt


def test_expected_weight_derivative_matches_corrected_appendix():
    """BC1: w_hat = sum sigma_n w_n; d w_hat / d d_n = (1/T) sigma_n (w_n - w_hat) (App. A Eq. devExtW
    with its n read as w_n = n/3), checked by finite differences."""
    rng = np.random.default_rng(3)
    d = torch.from_numpy(rng.standard_normal(4))
    Tt, wn = 0.3, torch.arange(4, dtype=torch.float64) / 3
    sig = torch.softmax(d / Tt, 0)
    what = (sig * wn).sum()
    analytic = sig * (wn - what) / Tt
    eps = 1e-6
    for n in range(4):
        dp, dm = d.clone(), d.clone()
        dp[n] += eps
        dm[n] -= eps
        fd = ((torch.softmax(dp / Tt, 0) * wn).sum() - (torch.softmax(dm / Tt, 0) * wn).sum()) / (2 * eps)
        assert abs(float(fd - analytic[n])) < 1e-8


def test_loss_closed_forms():
    """c_hat = c = a palette colour -> both loss terms vanish; the loss is a sum of squares (>= 0)."""
    e = torch.tensor([[0.2, 0.4, 0.6, 0.8, 0.6, 0.4]], dtype=torch.float64)
    pal = T.palettes(T.BC1, e)
    c = pal[:, 2]
    dec = T.ste_decoded(c, pal, 0.01)
    assert torch.allclose(dec, c)
    lay, params, xy, cref, eref, W, H = _setup([T.BC1, T.BC4])
    assert T.colour_loss(params, lay, [T.BC1, T.BC4], xy, W, H, cref, eref, 0.01) >= 0


def test_full_gradient_vs_finite_differences_of_the_surrogate():
    """With the STE the loss's gradient is that of the surrogate where c_dec is the softmax expectation
    in the backward pass only; at a large temperature we compare the autograd gradient of every
    parameter class against central differences of a loss whose c_dec is replaced by the hard value
    plus the (detached-free) expectation correction -- i.e. finite differences of
    L_c + 2 (hard - c) . soft  (same first derivative)."""
    fmts = [T.BC1, T.BC4]
    lay, params, xy, cref, eref, W, H = _setup(fmts, B=8)
    Tt = 2.0
    x = params.clone().requires_grad_(True)
    (g,) = torch.autograd.grad(T.colour_loss(x, lay, fmts, xy, W, H, cref, eref, Tt), x)

    def surrogate(p):
        # first-order model of the STE loss around the current hard decisions
        pp = T.unflatten(p, lay)
        u = (xy[:, 0].float() + 0.5) / W
        v = (xy[:, 1].float() + 0.5) / H
        a = T.grid_features([pp[f"grid{l}"] for l in range(2)], u, v)
        for l in range(3):
            a = torch.nn.functional.selu(a @ pp[f"W{l}"] + pp[f"b{l}"])
        chat = torch.sigmoid(a @ pp["W3"] + pp["b3"])
        with torch.no_grad():
            base = chat.clone()
        loss, co, eo = 0.0, 0, 0
        for f in fmts:
            w, we = (3, 6) if f == T.BC1 else (1, 2)
            pal = T.palettes(f, eref[:, eo:eo + we])
            ch, c = chat[:, co:co + w], cref[:, co:co + w]
            db = -torch.sqrt(((base[:, co:co + w][:, None] - pal) ** 2).sum(-1))
            hard = pal[torch.arange(pal.shape[0]), torch.argmax(db, 1)]
            d = -torch.sqrt(((ch[:, None] - pal) ** 2).sum(-1))
            soft = (torch.softmax(d / Tt, 1)[:, :, None] * pal).sum(1)
            loss = loss + ((ch - c) ** 2).sum() + (2 * (hard - c) * soft).sum()
            co, eo = co + w, eo + we
        return loss / xy.shape[0]

    rng = np.random.default_rng(4)
    n_grid = sum(int(np.prod(s)) for nme, s in lay if nme.startswith("grid"))
    idx = list(rng.choice(n_grid, 10, replace=False)) + list(n_grid + rng.choice(len(params) - n_grid, 30, replace=False))
    eps = 1e-6
    for i in idx:
        pp, pm = params.clone(), params.clone()
        pp[i] += eps
        pm[i] -= eps
        fd = (surrogate(pp) - surrogate(pm)) / (2 * eps)
        assert abs(float(fd) - float(g[i])) <= 1e-6 + 1e-5 * abs(float(g[i])), (i, float(fd), float(g[i]))


def test_adam_matches_torch_optim():
    rng = np.random.default_rng(5)
    p0 = torch.from_numpy(rng.standard_normal(50))
    m = torch.zeros(50, dtype=torch.float64)
    v = torch.zeros(50, dtype=torch.float64)
    ref = p0.clone().requires_grad_(True)
    opt = torch.optim.Adam([ref], lr=0.01, betas=(0.9, 0.999), eps=1e-15)
    p = p0.clone()
    for step in range(1, 4):
        g = torch.from_numpy(rng.standard_normal(50))
        p, m, v = T.adam(p, g, m, v, step, 0.01)
        ref.grad = g.clone()
        opt.step()
        assert torch.allclose(p, ref.detach(), rtol=1e-12, atol=1e-14)


def test_endpoint_gradient_vs_finite_differences_of_the_surrogate():
    """Endpoint network (Eq. 14): the autograd gradient of L_e + L_cd (STE) equals central
    differences of its first-order surrogate, in which the decoded colour is replaced by the softmax
    expectation over the REFERENCE palette weighted by 2 (hard - c), the distances taken against the
    PREDICTED palette."""
    fmts = [T.BC1, T.BC4]
    lay = T.layout_endpoint(fmts, 64, 2, 4)
    n = sum(int(np.prod(s)) for _, s in lay)
    rng = np.random.default_rng(6)
    params = torch.from_numpy(rng.standard_normal(n) * 0.3)
    B, BW, BH, Tt = 6, 16, 12, 2.0
    bxy = torch.from_numpy(np.stack([rng.integers(0, BW, B), rng.integers(0, BH, B)], 1))
    eref = torch.from_numpy(rng.uniform(0, 1, (B, 8)))
    c16 = torch.from_numpy(rng.uniform(0, 1, (B, 16, 4)))
    x = params.clone().requires_grad_(True)
    (g,) = torch.autograd.grad(T.endpoint_loss(x, lay, fmts, bxy, BW, BH, eref, c16, Tt), x)

    def ehat_of(p):
        pp = T.unflatten(p, lay)
        s = (bxy[:, 0].float() + 0.5) / BW
        t = (bxy[:, 1].float() + 0.5) / BH
        a = T.grid_features([pp["grid0"], pp["grid1"]], s, t)
        for l in range(3):
            a = torch.nn.functional.selu(a @ pp[f"W{l}"] + pp[f"b{l}"])
        return torch.sigmoid(a @ pp["W3"] + pp["b3"])

    base = ehat_of(params)

    def surrogate(p):
        eh = ehat_of(p)
        loss = ((eh - eref) ** 2).sum()
        eo = co = 0
        for f in fmts:
            w, we = (3, 6) if f == T.BC1 else (1, 2)
            pp_, pb = T.palettes(f, eh[:, eo:eo + we]), T.palettes(f, base[:, eo:eo + we])
            pr = T.palettes(f, eref[:, eo:eo + we])
            for i in range(16):
                c = c16[:, i, co:co + w]
                hard = pr[torch.arange(B), torch.argmin(((c[:, None] - pb) ** 2).sum(-1), 1)]
                d = -torch.sqrt(((c[:, None] - pp_) ** 2).sum(-1))
                soft = (torch.softmax(d / Tt, 1)[:, :, None] * pr).sum(1)
                loss = loss + (2 * (hard - c) * soft).sum()
            eo, co = eo + we, co + w
        return loss / B

    n_grid = sum(int(np.prod(s)) for nme, s in lay if nme.startswith("grid"))
    idx = list(rng.choice(n_grid, 8, replace=False)) + list(n_grid + rng.choice(n - n_grid, 24, replace=False))
    eps = 1e-6
    for i in idx:
        pp, pm = params.clone(), params.clone()
        pp[i] += eps
        pm[i] -= eps
        fd = (surrogate(pp) - surrogate(pm)) / (2 * eps)
        assert abs(float(fd) - float(g[i])) <= 1e-6 + 1e-5 * abs(float(g[i])), (i, float(fd), float(g[i]))


def test_qat_fake_quant_equals_inference_dequantization():
    """QAT (Eq. 1-5): the fake-quantized grid value is exactly what inference computes from the
    stored code (Eq. 2, the C oracle's o_dequant), the rounding error is at most s/2 inside the range,
    and the STE passes the gradient (1) only where the code is not clamped."""
    import oracle as O
    rng = np.random.default_rng(8)
    for lo, hi in ((-0.3, 0.7), (0.1, 0.2), (-1e-4, 1e-4)):
        g = torch.from_numpy(rng.uniform(lo, hi, (12, 12, 2))).requires_grad_(True)
        s, z = T.qat_params(g)
        q_val = T.fake_quant(g)
        r = T.round_half_away(g.detach().float() / s) + z
        codes = torch.clamp(r, 0, 255)
        deq = np.array([O.lib().o_dequant(int(c), float(s), int(z)) for c in codes.reshape(-1).tolist()], np.float32)
        assert np.array_equal(q_val.detach().float().reshape(-1).numpy(), deq)
        inside = (r == codes).reshape(-1).numpy()
        err = np.abs(q_val.detach().numpy().reshape(-1) - g.detach().numpy().reshape(-1))
        assert np.all(err[inside] <= float(s) * 0.5 * (1 + 1e-5) + 1e-12)
        (grad,) = torch.autograd.grad(q_val.sum(), g)
        assert np.array_equal(grad.reshape(-1).numpy(), inside.astype(np.float64))
    # half-way rounding: away from zero, exactly (the float32 floor(|x| + 1/2) shortcut fails at 0.49999997)
    x = torch.tensor([0.5, -0.5, 1.5, -2.5, 0.49999997, -0.49999997], dtype=torch.float32)
    assert T.round_half_away(x).tolist() == [1.0, -1.0, 2.0, -3.0, 0.0, -0.0]

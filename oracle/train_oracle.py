"""Training-step ORACLE for the NTBC colour network -- TEST INFRASTRUCTURE ONLY.

Plain PyTorch float64 on the CPU, autograd for the backward pass; only tests/ and bench-side tools
may import it.  Shares no code with the CUDA path.  One step follows PAPER.md:

  * features: the texel grid (fp32 master values, [res][res][2] per level, levels coarse -> fine) sampled
    at the texel centre exactly as at inference (R1-R3); optionally through the per-level
    8-bit fake quantizer of QAT (Eq. 1-5, the last 10% of training);
  * colour MLP 16 -> H -> H -> H -> N_c, selu hidden, sigmoid out, fp32 master weights;
  * loss L_color = L_c + L_cd (Eq. 14-15), per texel and texture:
      L_c  = |c_hat - c|^2,
      L_cd = |c_dec - c|^2 with c_dec the palette colour of the reference endpoints (Eq. 7/8) at
             n = argmax_n d_n, d_n = -|c_hat - c_n| (Eq. 9-10, colour-network case);
    averaged over the batch (R30);
  * STE through the argmax (App. A): forward uses c_dec, backward differentiates the
    expectation sum_n softmax(d/T)_n c_n (for BC1 this is (1 - w_hat) e0 + w_hat e1 with the expected
    weight w_hat of Eq. expected_weight; its derivative is (1/T) sigma_n (w_n - w_hat) -- App. A's
    Eq. devExtW prints "n - w_hat", a typo for w_n - w_hat); T = 0.01;
  * Adam, beta1 = 0.9, beta2 = 0.999, eps = 1e-15, separate learning rates for grids and MLP
    (P:341), bias-corrected as in Kingma & Ba.

Parameter vector layout (shared with the C ABI, R30): grid levels in order, each
[res][res][2] y-major; then per layer W [in][out] and b [out].
"""
from __future__ import annotations

import numpy as np
import torch

BC1, BC4 = 1, 4


def layout(fmts, hidden, levels, coarsest):
    """[(name, shape)] of the flat parameter vector."""
    n_c = sum(3 if f == BC1 else 1 for f in fmts)
    out = [(f"grid{l}", (coarsest << l, coarsest << l, 2)) for l in range(levels)]
    dims = [2 * levels, hidden, hidden, hidden, n_c]
    for l in range(4):
        out += [(f"W{l}", (dims[l], dims[l + 1])), (f"b{l}", (dims[l + 1],))]
    return out


def unflatten(vec, lay):
    parts, off = {}, 0
    for name, shape in lay:
        n = int(np.prod(shape))
        parts[name] = vec[off:off + n].reshape(shape)
        off += n
    return parts


def grid_features(grids, u, v):
    """Vertex-centred bilinear lookup per level (R1), concatenated coarse -> fine (R3).  The lattice
    coordinate is the inference convention (R1, R2): X = RN32(u (res - 1)) with u the binary32 texel
    centre, fx = X - floor(X) exactly; only the interpolation runs in float64."""
    feats = []
    u32, v32 = u.to(torch.float32), v.to(torch.float32)
    for g in grids:
        res = g.shape[0]
        X = u32 * torch.tensor(float(res - 1), dtype=torch.float32)
        Y = v32 * torch.tensor(float(res - 1), dtype=torch.float32)
        i0 = torch.clamp(torch.floor(X), max=res - 2).long()
        j0 = torch.clamp(torch.floor(Y), max=res - 2).long()
        fx, fy = (X - i0).double()[:, None], (Y - j0).double()[:, None]
        v00, v10 = g[j0, i0], g[j0, i0 + 1]
        v01, v11 = g[j0 + 1, i0], g[j0 + 1, i0 + 1]
        top = v00 + fx * (v10 - v00)
        bot = v01 + fx * (v11 - v01)
        feats.append(top + fy * (bot - top))
    return torch.cat(feats, dim=1)


def palettes(fmt, eref):
    """Palette colours [B][n][ch] of the reference endpoints (Eq. 7 / Eq. 8)."""
    if fmt == BC1:
        e0, e1 = eref[:, None, 0:3], eref[:, None, 3:6]
        w = torch.arange(4, dtype=eref.dtype)[None, :, None] / 3
        return (1 - w) * e0 + w * e1
    e0, e1 = eref[:, 0:1], eref[:, 1:2]
    m8 = (e0 > e1)
    w8 = torch.arange(8, dtype=eref.dtype)[None, :] / 7
    pal8 = (1 - w8) * e0 + w8 * e1
    w6 = (torch.arange(8, dtype=eref.dtype)[None, :] - 1) / 5
    pal6 = (1 - w6) * e0 + w6 * e1
    pal6 = torch.cat([torch.zeros_like(e0), pal6[:, 1:7], torch.ones_like(e0)], dim=1)
    return torch.where(m8, pal8, pal6)[:, :, None]


def ste_decoded(chat, pal, T):
    """c_dec in the forward pass, d(sum softmax(d/T) c_n) in the backward pass (App. A)."""
    diff = chat[:, None, :] - pal
    dist = torch.sqrt(torch.clamp((diff * diff).sum(-1), min=1e-30))   # |c_hat - c_n| (gradient-safe at 0)
    d = -dist
    n = torch.argmax(d, dim=1)                                          # first maximum: ties -> lower n
    hard = pal[torch.arange(pal.shape[0]), n]
    soft = (torch.softmax(d / T, dim=1)[:, :, None] * pal).sum(1)
    return soft + (hard - soft).detach()


def round_half_away(x):
    """Eq. 1's half-way rounding, read as round half away from zero (R33), exact in any precision:
    trunc(x) + sign(x) [|x - trunc(x)| >= 1/2]."""
    t = torch.trunc(x)
    return t + torch.sign(x) * (torch.abs(x - t) >= 0.5).to(x.dtype)


def qat_params(g):
    """Per-level asymmetric 8-bit quantizer parameters (Eq. 4-5, R4/R33) in binary32:
    s = (beta - alpha) / 255 from the level's min/max, z = round(-alpha / s)."""
    g32 = g.detach().to(torch.float32)
    alpha, beta = g32.min(), g32.max()
    s = (beta - alpha) / torch.tensor(255.0, dtype=torch.float32)
    z = round_half_away(-alpha / s) if float(s) > 0 else torch.zeros((), dtype=torch.float32)
    return s, z


def fake_quant(g):
    """Q(w) = s (clamp(round(w / s) + z; 0, 255) - z) (Eq. 3) evaluated in binary32 (as the stored
    int8 codes are dequantized at inference, Eq. 2); STE backward: 1 where not clamped, else 0 (P:174-178,
    whose printed "w" for the unclamped case is read as 1).  A constant level (s = 0) is left unchanged."""
    s, z = qat_params(g)
    if float(s) <= 0:
        return g
    g32 = g.detach().to(torch.float32)
    r = round_half_away(g32 / s) + z
    q = torch.clamp(r, 0.0, 255.0)
    mask = (r == q).to(g.dtype)
    deq = (s * (q - z)).to(g.dtype)
    return g * mask + (deq - g * mask).detach()


def _features(p, lay, levels, u, v, qat):
    grids = [p[f"grid{l}"] for l in range(levels)]
    if qat:
        grids = [fake_quant(g) for g in grids]
    return grid_features(grids, u, v)


def colour_loss(params, lay, fmts, xy, W, H, cref, eref, T, qat=False):
    p = unflatten(params, lay)
    levels = sum(1 for name, _ in lay if name.startswith("grid"))
    u = (xy[:, 0].float() + 0.5) / W           # binary32 texel centres (R2)
    v = (xy[:, 1].float() + 0.5) / H
    a = _features(p, lay, levels, u, v, qat)
    for l in range(3):
        a = torch.nn.functional.selu(a @ p[f"W{l}"] + p[f"b{l}"])
    chat = torch.sigmoid(a @ p["W3"] + p["b3"])
    loss = torch.zeros((), dtype=torch.float64)
    co = eo = 0
    for f in fmts:
        w, we = (3, 6) if f == BC1 else (1, 2)
        c, ch = cref[:, co:co + w], chat[:, co:co + w]
        dec = ste_decoded(ch, palettes(f, eref[:, eo:eo + we]), T)
        loss = loss + ((ch - c) ** 2).sum() + ((dec - c) ** 2).sum()
        co += w
        eo += we
    return loss / xy.shape[0]


def adam(params, grads, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-15):
    """One bias-corrected Adam update (Kingma & Ba): returns (params, m, v)."""
    m = beta1 * m + (1 - beta1) * grads
    v = beta2 * v + (1 - beta2) * grads * grads
    mh = m / (1 - beta1 ** step)
    vh = v / (1 - beta2 ** step)
    return params - lr * mh / (torch.sqrt(vh) + eps), m, v


def colour_step(params, m, v, step, lay, fmts, xy, W, H, cref, eref, T=0.01, lr_grid=0.01, lr_mlp=0.005, qat=False):
    """One training step; all arrays float64 torch tensors (xy int).  Returns (loss, grads, params, m, v)."""
    x = params.clone().requires_grad_(True)
    loss = colour_loss(x, lay, fmts, xy, W, H, cref, eref, T, qat)
    (g,) = torch.autograd.grad(loss, x)
    n_grid = sum(int(np.prod(s)) for name, s in lay if name.startswith("grid"))
    lr = torch.full_like(params, lr_mlp)
    lr[:n_grid] = lr_grid
    p2, m2, v2 = adam(params, g, m, v, step, lr)
    return float(loss.detach()), g, p2, m2, v2


# ---------------------------------------------------------------- endpoint network (Eq. 14)
def layout_endpoint(fmts, hidden, levels, coarsest):
    """Flat parameter vector of the endpoint network: block grid levels, then the MLP to N_e outputs."""
    n_e = sum(6 if f == BC1 else 2 for f in fmts)
    out = [(f"grid{l}", (coarsest << l, coarsest << l, 2)) for l in range(levels)]
    dims = [2 * levels, hidden, hidden, hidden, n_e]
    for l in range(4):
        out += [(f"W{l}", (dims[l], dims[l + 1])), (f"b{l}", (dims[l + 1],))]
    return out


def endpoint_loss(params, lay, fmts, bxy, BW, BH, eref, cref16, T, qat=False):
    """L_endpoint = L_e + L_cd (Eq. 14), batch mean.  eref [B][N_e] reference endpoints, cref16
    [B][16][N_c] reference colours of the block's texels (texel i = 4y + x).  The index of each texel
    comes from the PREDICTED endpoints' palette and the reference colour; the decoded colour is the
    REFERENCE endpoints' palette entry at that index; STE as for the colour network."""
    p = unflatten(params, lay)
    levels = sum(1 for name, _ in lay if name.startswith("grid"))
    s = (bxy[:, 0].float() + 0.5) / BW         # binary32 block centres (R2)
    t = (bxy[:, 1].float() + 0.5) / BH
    a = _features(p, lay, levels, s, t, qat)
    for l in range(3):
        a = torch.nn.functional.selu(a @ p[f"W{l}"] + p[f"b{l}"])
    ehat = torch.sigmoid(a @ p["W3"] + p["b3"])
    loss = ((ehat - eref) ** 2).sum()
    eo = co = 0
    B = bxy.shape[0]
    for f in fmts:
        w, we = (3, 6) if f == BC1 else (1, 2)
        pal_pred = palettes(f, ehat[:, eo:eo + we])            # [B][n][w], differentiable in ehat
        pal_ref = palettes(f, eref[:, eo:eo + we])
        for i in range(16):
            c = cref16[:, i, co:co + w]
            dist = torch.sqrt(torch.clamp(((c[:, None, :] - pal_pred) ** 2).sum(-1), min=1e-30))
            d = -dist
            n = torch.argmax(d, dim=1)
            hard = pal_ref[torch.arange(B), n]
            soft = (torch.softmax(d / T, dim=1)[:, :, None] * pal_ref).sum(1)
            dec = soft + (hard - soft).detach()
            loss = loss + ((dec - c) ** 2).sum()
        eo += we
        co += w
    return loss / B


def endpoint_step(params, m, v, step, lay, fmts, bxy, BW, BH, eref, cref16, T=0.01, lr_grid=0.01, lr_mlp=0.005,
                  qat=False):
    x = params.clone().requires_grad_(True)
    loss = endpoint_loss(x, lay, fmts, bxy, BW, BH, eref, cref16, T, qat)
    (g,) = torch.autograd.grad(loss, x)
    n_grid = sum(int(np.prod(s)) for name, s in lay if name.startswith("grid"))
    lr = torch.full_like(params, lr_mlp)
    lr[:n_grid] = lr_grid
    p2, m2, v2 = adam(params, g, m, v, step, lr)
    return float(loss.detach()), g, p2, m2, v2


# ---------------------------------------------------------------- test support: argmax decision margins
def _margin(dist):
    s, _ = torch.sort(dist, dim=1)
    return s[:, 1] - s[:, 0]


@torch.no_grad()
def colour_margins(params, lay, fmts, xy, W, H, eref, qat=False):
    """Per sample: the smallest gap between the nearest and second-nearest palette distance over the
    textures (float64).  Samples with a tiny gap can take the other argmax branch in fp32 arithmetic;
    parity tests drop them (the decision itself is discrete)."""
    p = unflatten(params, lay)
    levels = sum(1 for name, _ in lay if name.startswith("grid"))
    u = (xy[:, 0].float() + 0.5) / W           # binary32 texel centres (R2)
    v = (xy[:, 1].float() + 0.5) / H
    a = _features(p, lay, levels, u, v, qat)
    for l in range(3):
        a = torch.nn.functional.selu(a @ p[f"W{l}"] + p[f"b{l}"])
    chat = torch.sigmoid(a @ p["W3"] + p["b3"])
    m = torch.full((xy.shape[0],), float("inf"), dtype=torch.float64)
    co = eo = 0
    for f in fmts:
        w, we = (3, 6) if f == BC1 else (1, 2)
        pal = palettes(f, eref[:, eo:eo + we])
        dist = torch.sqrt(((chat[:, co:co + w][:, None] - pal) ** 2).sum(-1))
        m = torch.minimum(m, _margin(dist))
        co, eo = co + w, eo + we
    return m


@torch.no_grad()
def endpoint_margins(params, lay, fmts, bxy, BW, BH, cref16, qat=False):
    p = unflatten(params, lay)
    levels = sum(1 for name, _ in lay if name.startswith("grid"))
    s = (bxy[:, 0].float() + 0.5) / BW         # binary32 block centres (R2)
    t = (bxy[:, 1].float() + 0.5) / BH
    a = _features(p, lay, levels, s, t, qat)
    for l in range(3):
        a = torch.nn.functional.selu(a @ p[f"W{l}"] + p[f"b{l}"])
    ehat = torch.sigmoid(a @ p["W3"] + p["b3"])
    m = torch.full((bxy.shape[0],), float("inf"), dtype=torch.float64)
    eo = co = 0
    for f in fmts:
        w, we = (3, 6) if f == BC1 else (1, 2)
        pal = palettes(f, ehat[:, eo:eo + we])
        for i in range(16):
            dist = torch.sqrt(((cref16[:, i, co:co + w][:, None] - pal) ** 2).sum(-1))
            m = torch.minimum(m, _margin(dist))
        eo, co = eo + we, co + w
    return m

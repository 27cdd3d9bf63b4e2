"""Faithfulness accounting of north_star's agreement rule, shared by the CPU and GPU
faithfulness tests.  Test infrastructure: compares BC words / MLP outputs produced by any path (the
pinned oracle or the CUDA path) with those of the PLAIN-definition oracle (`oracle.plain_definitions`:
exact dot products, float64 libm activations, each rounded once).

Rule (BASELINE.json north_star):
  * floats: max |g - o| / |o| <= 1e-3 over all MLP outputs (o == 0 requires g == 0);
  * words: bit-exact, except a mismatched word is EXCUSED iff every differing field is explained by
    the plain oracle's value lying within 1e-4 of that field's decision boundary:
      - endpoint field: |e (2^b - 1) - (k + 1/2)| / (2^b - 1) < 1e-4 for the midpoint k + 1/2 between
        the two codes, which differ by one step (R11);
      - index field (endpoints equal): the texel's plain colour c lies within 1e-4 of the bisector of
        the two chosen palette entries, (|c - c_b|^2 - |c - c_a|^2) / (2 |c_a - c_b|) < 1e-4 (Eq.9-10);
  * reported by class: 5-bit / 6-bit / 8-bit endpoint, BC1 / BC4 index;
  * index ties: when the two chosen palette entries are EQUAL in exact arithmetic (Eq. 7/8 with the stored
    endpoints; e.g. a BC4 block with E0 == E1, whose 6-value entries 1..6 all equal E0/255 -- the binary32
    palette separates them only by rounding noise), both codes decode to the same value of the definition,
    so both are correct results (the order of equal keys); such words are counted as excused, class
    `index_tie`.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

import oracle

BC1, BC4 = 1, 4
BAND = 1e-4
# DirectX code -> linear palette index n (inverse of R16's maps)
_INV1 = {0: 0, 2: 1, 3: 2, 1: 3}
_INV4_8 = {0: 0, 2: 1, 3: 2, 4: 3, 5: 4, 6: 5, 7: 6, 1: 7}
_INV4_6 = {6: 0, 0: 1, 2: 2, 3: 3, 4: 4, 5: 5, 1: 6, 7: 7}
CLASSES = ("endpoint5", "endpoint6", "endpoint8", "index_bc1", "index_bc4", "index_tie")


def _exact_entry(fmt, hdr, n):
    """Palette entry n (linear order) in exact rational arithmetic (Eq. 7 / Eq. 8, UNORM endpoints)."""
    if fmt == BC1:
        c0, c1 = hdr & 0xFFFF, (hdr >> 16) & 0xFFFF
        e0 = [Fraction(c0 >> 11, 31), Fraction((c0 >> 5) & 63, 63), Fraction(c0 & 31, 31)]
        e1 = [Fraction(c1 >> 11, 31), Fraction((c1 >> 5) & 63, 63), Fraction(c1 & 31, 31)]
        w = Fraction(n, 3)
        return tuple((1 - w) * a + w * b for a, b in zip(e0, e1))
    E0, E1 = hdr & 0xFF, (hdr >> 8) & 0xFF
    e0, e1 = Fraction(E0, 255), Fraction(E1, 255)
    if E0 > E1:
        w = Fraction(n, 7)
    elif n == 0:
        return (Fraction(0),)
    elif n == 7:
        return (Fraction(1),)
    else:
        w = Fraction(n - 1, 5)
    return ((1 - w) * e0 + w * e1,)


def float_stats(g, o):
    """(max relative error over o != 0, max abs error, zero-violations, bit-exact fraction)."""
    g = np.asarray(g, np.float32).ravel()
    o = np.asarray(o, np.float32).ravel()
    zero = o == 0
    nz = ~zero
    rel = np.abs(g[nz].astype(np.float64) - o[nz]) / np.abs(o[nz].astype(np.float64))
    return {"max_rel": float(rel.max()) if rel.size else 0.0,
            "max_abs": float(np.max(np.abs(g.astype(np.float64) - o))) if g.size else 0.0,
            "zero_violations": int(np.count_nonzero(g[zero] != 0)),
            "bit_exact": float(np.mean(g.view(np.uint32) == o.view(np.uint32))) if g.size else 1.0}


def _near_mid(e: float, L: int, a: int, b: int) -> bool:
    if abs(a - b) != 1:
        return False
    return abs(float(e) * L - (min(a, b) + 0.5)) / L < BAND


def _ch565(c):
    return [(c >> 11) & 31, (c >> 5) & 63, c & 31]


def _endpoint_bc1(gw: int, pep6) -> tuple[str, bool]:
    """Header mismatch of a BC1 word: excused iff some assignment of the stored (swapped) endpoints to
    the predicted e0 / e1 differs from the plain codes only in near-midpoint channels."""
    Ls = [31, 63, 31]
    pc = [int(oracle.rgb565(pep6[0:3])), int(oracle.rgb565(pep6[3:6]))]
    pch = [_ch565(pc[0]), _ch565(pc[1])]
    gc = [gw & 0xFFFF, (gw >> 16) & 0xFFFF]
    cls, ok_any = None, False
    for g0, g1 in ((gc[0], gc[1]), (gc[1], gc[0])):
        gch = [_ch565(g0), _ch565(g1)]
        ok = True
        for e in range(2):
            for ch in range(3):
                if gch[e][ch] != pch[e][ch]:
                    cls = cls or ("endpoint6" if ch == 1 else "endpoint5")
                    ok &= _near_mid(pep6[3 * e + ch], Ls[ch], gch[e][ch], pch[e][ch])
        ok_any |= ok
    return cls or "endpoint5", ok_any


def _palette(fmt, hdr):
    if fmt == BC1:
        c0, c1 = hdr & 0xFFFF, (hdr >> 16) & 0xFFFF
        return oracle.palette_bc1(oracle.expand565(c0), oracle.expand565(c1)).astype(np.float64)
    E0, E1 = hdr & 0xFF, (hdr >> 8) & 0xFF
    return oracle.palette_bc4(E0, E1).astype(np.float64)[:, None]


def _index_excused(fmt, gw, pw, texels):
    """Index-only mismatch: every differing texel lies within 1e-4 of the bisector of the two entries, or
    the two entries are equal in exact arithmetic.  Returns (excused, all differences are such ties)."""
    if fmt == BC1:
        hdr, shift, bits, inv = pw & 0xFFFFFFFF, 32, 2, _INV1
    else:
        hdr, shift, bits = pw & 0xFFFF, 16, 3
        inv = _INV4_8 if (hdr & 0xFF) > ((hdr >> 8) & 0xFF) else _INV4_6
    pal = _palette(fmt, hdr)
    mask = (1 << bits) - 1
    tie = True
    for i in range(16):
        cg = (gw >> (shift + bits * i)) & mask
        cp = (pw >> (shift + bits * i)) & mask
        if cg == cp:
            continue
        if _exact_entry(fmt, hdr, inv[cp]) == _exact_entry(fmt, hdr, inv[cg]):
            continue   # equal entries of the definition: both codes are correct
        tie = False
        c = np.asarray(texels[i], np.float64).reshape(-1)
        a, b = pal[inv[cp]], pal[inv[cg]]
        sep = float(np.linalg.norm(a - b))
        if sep == 0.0:
            continue   # coincident entries: an exact tie
        dist = (float(np.sum((c - b) ** 2)) - float(np.sum((c - a) ** 2))) / (2.0 * sep)
        if not dist < BAND:
            return False, False
    return True, tie


def compare_words(fmts, gw, pw, pep, pcol, n_c_offsets=None, naive=False):
    """gw, pw: [tex][rows][BW] uint64 words (path under test, plain oracle); pep [rows][BW][N_e] and
    pcol [rows*4][W][N_c]: the plain oracle's MLP outputs of the same rows.  Returns a report dict:
    blocks, words, mismatched, excused, unexcused, and per-class counts."""
    assert not naive, "the excusal rule is stated for the NTBC colour network"
    n_tex = len(fmts)
    rows, BW = gw[0].shape
    rep = {"blocks": rows * BW, "words": rows * BW * n_tex, "mismatched": 0, "excused": 0, "unexcused": 0}
    for c in CLASSES:
        rep[c] = [0, 0]   # [excused, unexcused]
    eo = co = 0
    for k, f in enumerate(fmts):
        w = 3 if f == BC1 else 1
        g = np.asarray(gw[k]).view(np.uint64)
        p = np.asarray(pw[k]).view(np.uint64)
        for r, bx in np.argwhere(g != p):
            G, P = int(g[r, bx]), int(p[r, bx])
            e = pep[r, bx, eo:eo + 2 * w].astype(np.float64)
            hdr_mask = 0xFFFFFFFF if f == BC1 else 0xFFFF
            if (G & hdr_mask) != (P & hdr_mask):
                if f == BC1:
                    cls, ok = _endpoint_bc1(G, e)
                else:
                    cls = "endpoint8"
                    ok = True
                    for j, (gv, pv) in enumerate(((G & 0xFF, P & 0xFF), ((G >> 8) & 0xFF, (P >> 8) & 0xFF))):
                        if gv != pv:
                            ok &= _near_mid(e[j], 255, gv, pv)
            else:
                tex = [pcol[4 * r + (i >> 2), 4 * bx + (i & 3), co:co + w] for i in range(16)]
                ok, tie = _index_excused(f, G, P, tex)
                cls = "index_tie" if tie else "index_bc1" if f == BC1 else "index_bc4"
            rep["mismatched"] += 1
            rep["excused" if ok else "unexcused"] += 1
            rep[cls][0 if ok else 1] += 1
        eo += 2 * w
        co += w
    rep["excused_fraction_of_blocks"] = rep["excused"] / max(1, rep["blocks"])
    return rep

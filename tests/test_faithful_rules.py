"""Unit tests of the north_star agreement-rule accounting itself (tests/faithful.py, -m "not gpu"): each
excusal clause on hand-made words whose answer is known by construction."""
import numpy as np

import oracle
from faithful import BC1, BC4, _endpoint_bc1, _exact_entry, _index_excused, _near_mid, compare_words


def test_near_midpoint_rule():
    # e * 31 = 10.5 exactly: codes 10 and 11 are both one rounding away -> excused; 9 vs 11 never
    assert _near_mid(10.5 / 31, 31, 10, 11)
    assert _near_mid((10.5 + 31e-5) / 31, 31, 11, 10)            # 1e-5 (in [0,1] units) from the midpoint
    assert not _near_mid((10.5 + 31 * 2e-4) / 31, 31, 10, 11)    # 2e-4 away: outside the 1e-4 band
    assert not _near_mid(10.5 / 31, 31, 9, 11)


def test_bc1_endpoint_rule_follows_the_swap():
    """A BC1 header stores the endpoints in 4-colour order (c0 > c1, R12): the rule matches the stored codes
    to the predicted e0 / e1 in either order."""
    ep = np.array([10.5 / 31, 20 / 63, 5 / 31, 3 / 31, 40 / 63, 7 / 31])   # e0.r sits on a midpoint
    c0a = (10 << 11) | (20 << 5) | 5
    c0b = (11 << 11) | (20 << 5) | 5
    c1 = (3 << 11) | (40 << 5) | 7
    for c0 in (c0a, c0b):
        hi, lo = max(c0, c1), min(c0, c1)
        cls, ok = _endpoint_bc1(hi | (lo << 16), ep)
        assert ok
    far = ((12 << 11) | (20 << 5) | 5)                          # two codes away: unexcused
    cls, ok = _endpoint_bc1(max(far, c1) | (min(far, c1) << 16), ep)
    assert not ok and cls == "endpoint5"


def test_index_rule_bisector_and_exact_ties():
    # BC4 8-value block E0 = 200 > E1 = 100: entries n/7 apart; a texel exactly between entries 0 and 1
    E0, E1 = 200, 100
    pal = oracle.palette_bc4(E0, E1)
    mid = (float(pal[0]) + float(pal[1])) / 2
    hdr = E0 | (E1 << 8)
    code_n0, code_n1 = 0, 2                                    # linear 0 -> code 0, linear 1 -> code 2 (R16)
    w_plain = hdr | (code_n0 << 16)
    w_other = hdr | (code_n1 << 16)
    tex = [np.array([mid + 1e-6])] + [np.array([0.0])] * 15
    ok, tie = _index_excused(BC4, w_other, w_plain, tex)
    assert ok and not tie
    tex = [np.array([float(pal[0])])] + [np.array([0.0])] * 15   # on the entry itself: far from the bisector
    ok, tie = _index_excused(BC4, w_other, w_plain, tex)
    assert not ok
    # E0 == E1 (6-value mode): entries 1..6 are equal in exact arithmetic -> any of them is correct
    E = 52
    hdr = E | (E << 8)
    assert _exact_entry(BC4, hdr, 1) == _exact_entry(BC4, hdr, 4)
    ok, tie = _index_excused(BC4, hdr | (3 << 16), hdr | (0 << 16), [np.array([0.49])] * 16)   # codes 3 vs 0
    assert ok and tie


def test_compare_words_counts():
    fmts = [BC4]
    pal = oracle.palette_bc4(200, 100)
    mid = (float(pal[0]) + float(pal[1])) / 2
    hdr = 200 | (100 << 8)
    pw = np.array([[hdr]], np.uint64)
    gw = np.array([[hdr | (2 << 16)]], np.uint64)
    pep = np.array([[[200 / 255, 100 / 255]]], np.float32)
    pcol = np.zeros((4, 4, 1), np.float32)
    pcol[0, 0, 0] = mid
    rep = compare_words(fmts, [gw], [pw], pep, pcol)
    assert rep["mismatched"] == 1 and rep["excused"] == 1 and rep["index_bc4"] == [1, 0]
    pcol[0, 0, 0] = float(pal[0])
    rep = compare_words(fmts, [gw], [pw], pep, pcol)
    assert rep["unexcused"] == 1

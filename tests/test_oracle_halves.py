"""Pins of the oracle's "halves" indicator layout (R26, DSI_F_RNG_HALVES).

The layout must equal its plain definition -- one 32-bit comparison of the concatenation
(v << 16 | w) with thr, v and w the 16-bit halves named by the layout and drawn from the
KAT-pinned Philox -- and give the Bernoulli(thr / 2^32) law, including thresholds where every
acceptance (or every rejection) comes through a tie (v == T).  The oracle evaluates the lazy
three-way comparison (v < T, v > T, tie-break); these tests never call that code path's helpers.
"""
import numpy as np
import pytest

import oracle as O

SEED = 0x5EED_2405_1410_5
KEY = (SEED & 0xFFFFFFFF, SEED >> 32)


def indicators(a, trial, n_pos, stream=0):
    """A_1..A_n from the oracle (acc of N = p+1 minus acc of N = p)."""
    acc = [0]
    for p in range(1, n_pos + 1):
        c = O.Config(1, 1, a, 1, 1, p + 1, stream, rng_halves=True)
        acc.append(O.trial(c, SEED, trial)["acc"])
    return [acc[p] - acc[p - 1] for p in range(1, n_pos + 1)]


def half(words, j):
    """The layout's 16-bit draw for offset j: high half of word j (j < 4), low half of word j-4."""
    w = words[j % 4]
    return (w >> 16) if j < 4 else (w & 0xFFFF)


def concatenated(thr, trial, p, stream=0):
    q, j = (p - 1) // 8, (p - 1) % 8
    v = half(O.philox4x32_10((q, 0, trial, stream), KEY), j)
    w = half(O.philox4x32_10((q, 1, trial, stream), KEY), j)
    return int(((v << 16) | w) < thr), v


@pytest.mark.parametrize("a", [0.8, 0.3, 0.5 - 2 ** -20, 2 ** -17, 1 - 2 ** -17])
def test_halves_equal_the_concatenated_comparison(a):
    thr = O.threshold(a)
    for trial in (0, 1, 77):
        got = indicators(a, trial, 40, stream=trial % 3)
        want = [concatenated(thr, trial, p, stream=trial % 3)[0] for p in range(1, 41)]
        assert got == want, (a, trial)


@pytest.mark.parametrize("j", range(8))
@pytest.mark.parametrize("side", ["accept", "reject"])
def test_forced_ties_take_the_tie_break(j, side):
    """thr chosen so that the draw at offset j of call 0 ties (v == T): A_p is then [w < R]."""
    trial, p = 5, j + 1
    v = half(O.philox4x32_10((0, 0, trial, 0), KEY), j)
    w = half(O.philox4x32_10((0, 1, trial, 0), KEY), j)
    R = min(w + 1, 0xFFFF) if side == "accept" else w  # accept needs w < R, reject w >= R
    if side == "accept" and w == 0xFFFF:
        pytest.skip("w = 0xFFFF cannot be accepted at a tie")
    thr = (v << 16) | R
    a = thr / 2 ** 32  # exact: thr < 2^32
    assert O.threshold(a) == thr
    got = indicators(a, trial, p)[p - 1]
    assert got == (1 if side == "accept" else 0)
    assert got == concatenated(thr, trial, p)[0]


@pytest.mark.parametrize("thr", [0x8000, 0xFFFF8000, 0x4CCCCCCC, 0x80000000])
def test_halves_law(thr):
    """Acceptance frequency within 6 sigma of thr / 2^32 over 2.4e6 positions, including thr <
    2^16 (T = 0: every acceptance is a tie) and T = 0xFFFF (every rejection is a tie)."""
    a = thr / 2 ** 32
    N, T = 1201, 2000
    r = O.run(O.Config(1, 1, a, 1, 1, N, 0, rng_halves=True), SEED, 0, T)
    n = (N - 1) * T
    mean = r["sum_acc"] / n
    sd = (a * (1 - a) / n) ** 0.5
    assert abs(mean - a) <= 6 * sd + 1e-12, (thr, mean, a)
    if thr < 0x10000:
        assert r["sum_acc"] > 0  # ties are the only way to accept here


def test_halves_and_words_share_the_law_but_not_the_draws():
    c = O.Config(10, 1, 0.6, 4, 3, 300, 1)
    a = O.run(c, SEED, 0, 400)
    b = O.run(O.Config(10, 1, 0.6, 4, 3, 300, 1, rng_halves=True), SEED, 0, 400)
    assert a["sum_acc"] != b["sum_acc"]
    n = 299 * 400
    assert abs(a["sum_acc"] - b["sum_acc"]) / n < 6 * (2 * 0.24 / n) ** 0.5


def test_halves_degenerate_thresholds():
    for a, want in ((0.0, 0), (1.0, 1)):
        r = O.run(O.Config(3, 1, a, 2, 2, 64, 0, rng_halves=True), SEED, 0, 50)
        assert r["sum_acc"] == want * 63 * 50


@pytest.mark.parametrize("j", [1, 2, 3])
def test_multi_drafter_halves_equal_the_concatenated_comparison(j):
    """The multi-drafter oracle's halves indicator (drafter j on counter word 1 = 2(j-1), its
    tie-break on 2(j-1)+1) equals the plain 32-bit comparison of the concatenated halves."""
    rates = (0.8, 0.49, 2.0 ** -17)
    cfg = O.MultiConfig(100, (2, 5, 9), rates, 50, 1, rng_halves=True)
    thr = O.threshold(rates[j - 1])
    for trial in (0, 9):
        for p in range(1, 41):
            q, j8 = (p - 1) // 8, (p - 1) % 8
            v = half(O.philox4x32_10((q, 2 * (j - 1), trial, 1), KEY), j8)
            w = half(O.philox4x32_10((q, 2 * (j - 1) + 1, trial, 1), KEY), j8)
            assert O.multi_indicator(cfg, SEED, trial, j, p) == int(((v << 16) | w) < thr), (j, trial, p)


def test_multi_drafter_halves_drafter1_is_the_single_drafter_stream():
    a = 0.49
    cfg = O.MultiConfig(100, (5,), (a,), 41, 0, rng_halves=True)
    got = [O.multi_indicator(cfg, SEED, 4, 1, p) for p in range(1, 41)]
    assert got == indicators(a, 4, 40)

"""Pins of the oracle's TTFT variant ("generating the first
token adds a wait of TTFT while generating each subsequent token adds a wait of TPOT").
Reading (R23): the first forward of each model costs its TTFT -- the drafter's
first draft and the target pool's first-ever forward (thread 0 of the first segment),
as in SPEC S:96."""
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import exact_math as X

SEED = 2405141050


def test_nonsi_examples_of_spec():
    # (ttft 50, tpot 30, N = 1) -> 50 ms; (ttft 100, tpot 20.6, N = 50) -> 1109.4 ms
    r = O.trial(O.Config(30, 6, 0.5, 1, 2, 1, t_target_first=50), SEED, 0)
    assert r["nonsi"] == 50
    r = O.trial(O.Config(206, 68, 0.5, 1, 8, 50, t_target_first=1000, t_drafter_first=80), SEED, 0)
    assert r["nonsi"] == 11094  # ticks of 0.1 ms


def test_hand_examples():
    # a = 0, k = 1, N = 3, t_d 1, t_t 10, first forwards 3 and 25:
    # SI: (3 + 25) + 11 + 11 = 50; DSI: 25 + 10 + 10 = 45 = non-SI (Thm 1 equality case)
    cfg = O.Config(10, 1, 0.0, 1, 1, 3, t_target_first=25, t_drafter_first=3)
    r = O.trial(cfg, SEED, 0)
    assert (r["si"], r["dsi"], r["nonsi"]) == (50, 45, 45)
    # a = 1, k = 1, one server: every forward queues behind the first -> DSI = non-SI
    cfg = O.Config(100, 14, 1.0, 1, 1, 9, t_target_first=300, t_drafter_first=40)
    r = O.trial(cfg, SEED, 0)
    assert r["dsi"] == 300 + 8 * 100 == r["nonsi"]
    # a = 1, k = 1, enough servers: the last thread is requested at t_d1 + (N-2) t_d,
    # but position 1 is only settled at t_t1
    for t_t1 in (120, 2000):
        cfg = O.Config(100, 14, 1.0, 1, 16, 12, t_target_first=t_t1, t_drafter_first=40)
        assert O.trial(cfg, SEED, 0)["dsi"] == max(t_t1, 40 + 10 * 14 + 100)


@pytest.mark.parametrize("N,k,sp,t_d,t_t,t_t1,t_d1", [
    (9, 1, 2, 14, 100, 536, 15), (10, 2, 3, 7, 50, 62, 9), (8, 3, 1, 10, 30, 300, 12),
    (11, 1, 16, 5, 40, 400, 6), (7, 5, 2, 3, 20, 21, 3), (10, 2, 2, 30, 100, 160, 30)])
def test_enumeration_matches_exact_expectation(N, k, sp, t_d, t_t, t_t1, t_d1):
    """All 2^(N-1) patterns through the event simulation vs the exact expectation built from
    an independent FIFO schedule of the first segment (incl. out-of-order completions)."""
    a = Fraction(2, 3)
    cfg = O.Config(t_t, t_d, 0.5, k, sp, N, t_target_first=t_t1, t_drafter_first=t_d1)
    r = O.run(cfg, SEED, 0, 1 << (N - 1), pattern=True)

    def per(A):
        i = X.pattern_index(A)
        return {"dsi": int(r["dsi"][i]), "si": int(r["si"][i])}

    got = X.enumerate_expectations(N, a, per)
    want = X.expectations_ttft(N, k, t_d, t_t, sp, a, t_t1, t_d1)
    assert got["dsi"] == want["dsi"] and got["si"] == want["si"]


def test_ttft_equal_to_tpot_is_the_base_model():
    rng = random.Random(9)
    for _ in range(30):
        t_t = rng.randint(2, 100)
        t_d = rng.randint(1, t_t)
        base = O.Config(t_t, t_d, rng.random(), rng.randint(1, 8), rng.randint(1, 8), rng.randint(1, 50))
        same = O.Config(*[getattr(base, f) for f in ("t_target", "t_drafter", "accept_rate", "lookahead",
                                                     "sp_degree", "n_tokens", "stream_id")],
                        t_target_first=t_t, t_drafter_first=t_d)
        a, b = O.run(base, SEED, 0, 20), O.run(same, SEED, 0, 20)
        for key in ("si", "dsi", "iters", "acc"):
            assert np.array_equal(a[key], b[key])


def test_theorem1_with_ttft():
    """DSI <= non-SI per trial when k t_d <= t_t and the first forwards obey t_d1 <= t_t1."""
    rng = random.Random(10)
    for _ in range(120):
        t_t = rng.randint(2, 120)
        t_d = rng.randint(1, t_t)
        k = rng.randint(1, max(1, t_t // t_d))
        t_t1 = rng.randint(t_t, 6 * t_t)
        t_d1 = rng.randint(1, min(t_t1, 6 * t_d))
        cfg = O.Config(t_t, t_d, rng.choice([0.0, 1.0, rng.random()]), k, rng.randint(1, 8),
                       rng.randint(1, 60), t_target_first=t_t1, t_drafter_first=t_d1)
        r = O.run(cfg, SEED, rng.randint(0, 999), 10)
        assert r["n_dsi_gt_nonsi"] == 0, cfg

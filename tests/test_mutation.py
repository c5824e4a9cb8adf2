"""Mutation test ("a deliberately wrong C(g) must fail parity"; SPEC's test-only
--inject-skip-cancel idea): libdsi_sim_mutant.so is built from the same sources with
-DDSI_MUTANT_CG, which makes every DSI segment cost C(g), g >= 2, one tick too large
(dsi_common.cuh seg_extra).  The parity checks used everywhere else must catch it: the mutant's
per-trial L_DSI and sums differ from the oracle, the product's do not.  Also a CPU check that
the oracle's pins catch a wrong cost: Table 1 computed with C(g) + 1 no longer matches."""
import numpy as np
import pytest

import oracle as O

from helpers import oracle_sums

D = pytest.importorskip("paper_2405_14105_b200.dsi_sim")
from paper_2405_14105_b200 import workloads as W  # noqa: E402

SEED = W.SEED


def _dsi_trials(variant, cfgs, tick):
    with D.use_library(variant):
        with D.Simulator(cfgs, tick=tick, seed=SEED, flags=D.DSI_F_PER_TRIAL) as sim:
            sim.run()
            res = sim.reduce()
            return res, [sim.trials(i)["dsi"].astype(np.int64) for i in range(len(cfgs))]


@pytest.mark.gpu
def test_parity_catches_a_wrong_segment_cost():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfgs, tick = W.cfg1(trials=1000)
    fz, ftick = W.fuzz(40, seed=11, trials=200)
    for c, t in ((cfgs, tick), (fz, ftick)):
        want = [oracle_sums(row, t, SEED, hist=False, per_trial=True) for row in c]
        res, got = _dsi_trials("product", c, t)
        assert all(np.array_equal(g, w["dsi"]) for g, w in zip(got, want))
        assert all(int(r["sum_dsi_ticks"]) == w["sum_dsi"] for r, w in zip(res, want))
        mres, mgot = _dsi_trials("mutant", c, t)
        bad = sum(not np.array_equal(g, w["dsi"]) for g, w in zip(mgot, want))
        bad_sums = sum(int(r["sum_dsi_ticks"]) != w["sum_dsi"] for r, w in zip(mres, want))
        # every config with a segment of length >= 2 in some trial is caught, by trial and by sum
        assert bad >= 1 and bad_sums >= 1, (bad, bad_sums)
        for g, w, r, row in zip(mgot, want, mres, c):
            # the mutant differs exactly by the number of g >= 2 segments: never silently equal
            n2 = g - w["dsi"]
            assert (n2 >= 0).all() and int(r["sum_dsi_ticks"]) - w["sum_dsi"] == int(n2.sum())


def _half(words, j):
    w = words[j % 4]
    return (w >> 16) if j < 4 else (w & 0xFFFF)


@pytest.mark.gpu
def test_halves_parity_catches_a_dropped_tie_break():
    """The mutant also drops the halves layout's tie-break (-DDSI_MUTANT_TIES: ties stay
    rejections).  On thresholds built so that chosen positions tie and the tie-break accepts, the
    per-trial accept counts -- which the C(g) mutation does not touch -- must differ from the
    oracle's with the mutant and equal them with the product."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    key = (SEED & 0xFFFFFFFF, SEED >> 32)
    rows = []
    for q, j in ((0, 0), (0, 5), (1, 3), (6, 7), (12, 2)):
        v = _half(O.philox4x32_10((q, 0, 0, 0), key), j)
        w = _half(O.philox4x32_10((q, 1, 0, 0), key), j)
        if w < 0xFFFF:
            rows.append((1.0, 0.2, ((v << 16) | (w + 1)) / 2 ** 32, 3, 3, 100, 0, 40))  # tie, accepted
    cfgs = W.rows(rows)
    want = [oracle_sums(row, 0.01, SEED, per_trial=True, halves=True) for row in cfgs]
    for variant in ("product", "mutant"):
        with D.use_library(variant):
            with D.Simulator(cfgs, tick=0.01, seed=SEED, flags=D.DSI_F_PER_TRIAL | D.DSI_F_RNG_HALVES) as sim:
                sim.run()
                sim.reduce()
                acc = [sim.trials(i)["acc"].astype(np.int64) for i in range(len(cfgs))]
        same = [np.array_equal(a, w["acc"]) for a, w in zip(acc, want)]
        if variant == "product":
            assert all(same)
        else:  # trial 0 ties at the chosen position in every config
            assert not any(same)
            assert all(int(a[0]) == int(w["acc"][0]) - 1 for a, w in zip(acc, want))


def test_oracle_pins_catch_a_wrong_segment_cost():
    """CPU: which oracle pins would catch C(g) + 1.  Prop. 1's per-trial identity (P:211-213,
    L_DSI = t_d acc + t_t (N - acc) at k = 1 with enough servers) does, on every trial that has a
    segment of length >= 2, and the oracle's event simulation satisfies it; Table 1
    does NOT -- its instants sit in 14-tick windows (R22), so a one-tick slip leaves every count
    unchanged, which is why the per-trial parity above is the check that matters."""
    import json
    import os
    import random
    import exact_math as X
    t_t, t_d, k, sp = 100, 14, 1, 8
    rng = random.Random(3)
    caught = 0
    for _ in range(200):
        N = rng.randint(2, 33)
        A = [int(rng.random() < 0.7) for _ in range(N - 1)]
        prop1 = t_d * sum(A) + t_t * (N - sum(A))
        lit = O.trial(O.Config(t_t, t_d, 0.5, k, sp, N), SEED, X.pattern_index(A), pattern=True)["dsi"]
        mutated = sum(X.C(g, k, t_d, t_t, sp) + (g >= 2) for g in X.segments(A, N))
        assert lit == prop1
        caught += mutated != prop1
        assert (mutated != prop1) == any(g >= 2 for g in X.segments(A, N))
    assert caught > 150
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")))

    def count(t, cost):  # max n with L(N = n) <= t, every draft accepted: one segment of length n
        return max(n for n in range(1, 200) if cost(n) <= t)

    bad = [count(t, lambda n: X.C(n, 1, 14, 100, 7) + (n >= 2)) for t in g["times"]]
    assert bad == g["best_case"]["dsi"]  # the documented blind spot of the Table 1 pin

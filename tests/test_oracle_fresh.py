"""Pins of the oracle's fresh-verifier variant (R24).

Thm 2's proof lets DSI "invoke a new current verifier thread" when the verifier
accepts; Alg. 1 line 10 terminates the verifier's own child, so the default
model (R5) has no such thread and can lose to non-SI and SI when k t_d > t_t.  The
variant starts a fresh target forward whenever the committed prefix grows and no
started thread would settle the next position within t_t.  Pinned by: hand-derived
schedules (tests/golden/fresh_verifier.json), an independent closed form derived by hand
(exact_math.C_fresh) over every pattern of small N, identity with the default model when
k t_d <= t_t, Thm 1 per trial for every (k, SP), the bound of Thm 2's proof
 and Thm 2 per coupled trial under Eq. 1."""
import json
import os
import random
from fractions import Fraction

import pytest

import oracle as O
import exact_math as X

SEED = 2405141050
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "fresh_verifier.json")


def cfg(t_t, t_d, a, k, sp, N, fresh=True, **kw):
    return O.Config(t_t, t_d, a, k, sp, N, fresh_verifier=fresh, **kw)


def test_golden_hand_schedules():
    g = json.load(open(GOLDEN))["examples"]
    e = g[0]
    for N, (want, want_default) in enumerate(zip(e["dsi_by_n_tokens"], e["default_dsi_by_n_tokens"]), 1):
        c = (e["t_target"], e["t_drafter"], 1.0, e["lookahead"], e["sp_degree"], N)
        assert O.trial(cfg(*c), SEED, 0)["dsi"] == want, N
        assert O.trial(cfg(*c, fresh=False), SEED, 0)["dsi"] == want_default, N
    e = g[1]
    c = (e["t_target"], e["t_drafter"], 0.5, e["lookahead"], e["sp_degree"], e["n_tokens"])
    i = X.pattern_index(e["A"])
    r = O.trial(cfg(*c), SEED, i, pattern=True)
    assert (r["dsi"], r["si"], r["nonsi"]) == (e["dsi"], e["si"], e["nonsi"])
    assert O.trial(cfg(*c, fresh=False), SEED, i, pattern=True)["dsi"] == e["default_dsi"]


def test_event_simulation_matches_hand_closed_form_on_every_pattern():
    rng = random.Random(11)
    cases = [(10, 4, 5, 1, 12), (100, 14, 20, 7, 12), (30, 30, 3, 2, 11), (7, 2, 9, 3, 12)]
    cases += [(rng.randint(1, 40), 0, rng.randint(1, 12), rng.randint(1, 6), rng.randint(1, 10))
              for _ in range(40)]
    for t_t, t_d, k, sp, N in cases:
        t_d = t_d or rng.randint(1, t_t)
        r = O.run(cfg(t_t, t_d, 0.5, k, sp, N), SEED, 0, 1 << (N - 1), pattern=True)
        for i in range(1 << (N - 1)):
            A = [(i >> p) & 1 for p in range(N - 1)]
            assert int(r["dsi"][i]) == X.closed_form_fresh(A, N, k, t_d, t_t, sp)["dsi"], \
                (t_t, t_d, k, sp, N, A)


def test_identical_to_default_when_k_td_le_tt():
    rng = random.Random(5)
    for _ in range(150):
        t_t = rng.randint(1, 120)
        t_d = rng.randint(1, t_t)
        k = rng.randint(1, max(1, t_t // t_d))
        sp, N = rng.randint(1, 8), rng.randint(1, 90)
        a = rng.choice([0.0, 1.0, rng.random()])
        assert k * t_d <= t_t
        f = O.run(cfg(t_t, t_d, a, k, sp, N), SEED, 0, 30)
        d = O.run(cfg(t_t, t_d, a, k, sp, N, fresh=False), SEED, 0, 30)
        assert list(f["dsi"]) == list(d["dsi"]) and list(f["si"]) == list(d["si"])


def test_theorem1_per_trial_for_every_lookahead():
    """P:199-201 (DSI is never slower than non-SI): each position settles within t_t of its
    predecessor, so L_DSI <= N t_t for every k and SP -- also where the default model
    breaks it (k t_d > t_t, R5)."""
    rng = random.Random(9)
    broke_default = 0
    for _ in range(200):
        t_t = rng.randint(1, 60)
        t_d = rng.randint(1, t_t)
        k, sp, N = rng.randint(1, 24), rng.randint(1, 8), rng.randint(1, 80)
        a = rng.choice([0.0, 1.0, rng.random(), rng.random()])
        f = O.run(cfg(t_t, t_d, a, k, sp, N), SEED, 0, 25)
        assert f["n_dsi_gt_nonsi"] == 0
        broke_default += O.run(cfg(t_t, t_d, a, k, sp, N, fresh=False), SEED, 0, 25)["n_dsi_gt_nonsi"]
    assert broke_default > 0  # the fuzz does reach the cases the variant exists for


@pytest.mark.parametrize("t_t,t_d,k", [(10, 4, 5), (100, 14, 20), (100, 100, 3), (50, 7, 8), (9, 9, 1)])
def test_bound_of_theorem2_proof(t_t, t_d, k):
    """if the first k drafts are accepted (n = k), x_{k+1} is committed at
    k t_1 + t_2 and DSI completes x_{k+2} at time <= k t_1 + 2 t_2 (over at least
    ceil(t_2/(k t_1)) servers).  N = k + 2 with a = 1: exactly k t_d + t_t + min(k t_d, t_t)."""
    sp = -(-t_t // (k * t_d))
    r = O.trial(cfg(t_t, t_d, 1.0, k, sp, k + 2), SEED, 0)
    assert r["dsi"] <= k * t_d + 2 * t_t
    assert r["dsi"] == k * t_d + t_t + min(k * t_d, t_t)


def test_theorem2_per_coupled_trial_under_eq1():
    """with Eq. 1 (ceil(t_t/(k t_d)) <= SP), L_DSI <= L_SI on every coupled trial
    at equal k -- the default model meets it only when k t_d <= t_t (R6)."""
    rng = random.Random(13)
    broke_default = 0
    for _ in range(200):
        t_t = rng.randint(1, 60)
        t_d = rng.randint(1, t_t)
        k, N = rng.randint(1, 24), rng.randint(1, 80)
        sp = -(-t_t // (k * t_d)) + rng.randint(0, 3)
        a = rng.choice([0.0, 1.0, rng.random(), rng.random()])
        f = O.run(cfg(t_t, t_d, a, k, sp, N), SEED, 0, 25)
        assert f["n_dsi_gt_si"] == 0
        broke_default += O.run(cfg(t_t, t_d, a, k, sp, N, fresh=False), SEED, 0, 25)["n_dsi_gt_si"]
    assert broke_default > 0


@pytest.mark.parametrize("N,k,sp,t_d,t_t", [(10, 5, 1, 4, 10), (12, 20, 7, 14, 100), (9, 3, 2, 30, 40),
                                            (11, 2, 3, 11, 12)])
def test_enumeration_matches_exact_expectation(N, k, sp, t_d, t_t):
    a = Fraction(3, 5)
    r = O.run(cfg(t_t, t_d, 0.5, k, sp, N), SEED, 0, 1 << (N - 1), pattern=True)
    got = X.enumerate_expectations(N, a, lambda A: {"dsi": int(r["dsi"][X.pattern_index(A)])})
    assert got["dsi"] == X.expectations_fresh(N, k, t_d, t_t, sp, a)["dsi"]


def test_not_with_ttft():
    with pytest.raises(Exception):
        O.trial(cfg(10, 4, 0.5, 5, 1, 8, t_target_first=20), SEED, 0)

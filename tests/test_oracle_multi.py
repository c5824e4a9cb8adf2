"""Pins of the multi-drafter oracle (R25): Algorithm 1 with m > 2
models, lookahead 1, unbounded threads.

Two oracle forms: the literal thread tree (every finished thread spawns m children, the
verifier terminates and relabels; exponential) and the verified-chain simulation (linear).
Pinned by: hand-traced trees (tests/golden/multi_drafter.json), Prop. 1 when m = 2
 and identity with the single-drafter event simulation at k = 1, Thm 1 per trial
(proof P:418), exhaustive enumeration of all m^(N-1) outcome patterns against
exact rational expectations, and monotonicity in the drafter set (appending a drafter that
is slower than every other drafter can only settle positions sooner)."""
import json
import os
import random
from fractions import Fraction

import pytest

import oracle as O

SEED = 2405141050
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "multi_drafter.json")


def pattern_index(j_star, m):
    """Trial index of the enumeration mode: digit p-1 in base m is j*(p) - 1."""
    i = 0
    for p, j in enumerate(j_star):
        i += (j - 1) * m ** p
    return i


def test_golden_hand_traced_trees():
    for e in json.load(open(GOLDEN))["examples"]:
        m = len(e["t_drafters"]) + 1
        c = O.MultiConfig(e["t_target"], tuple(e["t_drafters"]), (0.5,) * (m - 1), e["n_tokens"])
        i = pattern_index(e["j_star"], m)
        for r in (O.multi_tree(c, SEED, i, pattern=True), O.multi_chain(c, SEED, i, pattern=True)):
            assert (r["dsi"], r["nonsi"], r["settled"]) == (e["dsi"], e["nonsi"], e["settled"]), e["name"]


def test_pattern_indicators_follow_j_star():
    c = O.MultiConfig(10, (2, 5), (0.5, 0.5), 4)
    i = pattern_index([1, 3, 2], 3)
    got = [[O.multi_indicator(c, SEED, i, j, p, pattern=True) for p in (1, 2, 3)] for j in (1, 2)]
    assert got == [[1, 0, 0], [1, 0, 1]]


def test_drafter_one_draws_the_single_drafter_stream():
    """Counter word 1 is j-1, so drafter 1 sees exactly the indicators of the single-drafter
    contract (counter (q, 0, trial, stream)); drafter 2 is the same generator at word 1 = 1."""
    rng = random.Random(3)
    for _ in range(30):
        a1, a2 = rng.random(), rng.random()
        N, trial, stream = rng.randint(2, 40), rng.randrange(1 << 32), rng.randrange(1 << 32)
        c = O.MultiConfig(100, (10, 20), (a1, a2), N, stream)
        acc = sum(O.multi_indicator(c, SEED, trial, 1, p) for p in range(1, N))
        single = O.trial(O.Config(100, 10, a1, 1, 1, N, stream), SEED, trial)
        assert acc == single["acc"]
        key = (SEED & 0xFFFFFFFF, SEED >> 32)
        for p in range(1, N):
            u = O.philox4x32_10(((p - 1) >> 2, 1, trial, stream), key)[(p - 1) & 3]
            assert O.multi_indicator(c, SEED, trial, 2, p) == int(u < O.threshold(a2))


def test_two_models_equal_single_drafter_event_simulation():
    """m = 2 is the single-drafter model at k = 1 with SP >= ceil(t_t/t_d) (no queueing), whose
    DSI latency is Prop. 1 per trial -- same indicators, same latency."""
    rng = random.Random(7)
    for _ in range(25):
        t_t = rng.randint(1, 60)
        t_d = rng.randint(1, t_t)
        a, N = rng.random(), rng.randint(1, 30)
        sp = -(-t_t // t_d)
        c = O.MultiConfig(t_t, (t_d,), (a,), N)
        single = O.run(O.Config(t_t, t_d, a, 1, sp, N), SEED, 0, 40)
        multi = O.multi_run(c, SEED, 0, 40)
        assert list(multi["dsi"]) == list(single["dsi"])
        assert [int(s[0]) for s in multi["settled"]] == list(single["acc"])
        for t in range(0, 40, 8):
            if N <= 12:
                assert O.multi_tree(c, SEED, t)["dsi"] == int(single["dsi"][t])


CASES = [
    (10, (2, 5), 6), (10, (4, 10), 6), (7, (1, 2, 3), 5), (12, (3, 3), 6), (5, (5,), 9),
    (9, (1, 4, 6, 9), 4), (20, (2, 7, 11), 5),
]


@pytest.mark.parametrize("t_t,t_ds,N", CASES)
def test_tree_equals_chain_on_every_pattern_and_exact_expectation(t_t, t_ds, N):
    """Every one of the m^(N-1) outcome patterns through the literal thread tree and the chain
    simulation; the pattern-weighted mean equals the exact expectation
    E[L] = t_m + (N-1) sum_j t_j pi_j, pi_j = a_j prod_{i<j}(1-a_i) (linearity over positions,
    each position's j* i.i.d. with law pi, P:418 + P:423)."""
    m = len(t_ds) + 1
    rates = [Fraction(1, 3), Fraction(3, 5), Fraction(1, 2), Fraction(2, 7), Fraction(4, 5)][:m - 1]
    c = O.MultiConfig(t_t, t_ds, tuple(float(a) for a in rates), N)
    pi = []
    rest = Fraction(1)
    for a in rates:
        pi.append(rest * a)
        rest *= 1 - a
    pi.append(rest)
    lat = list(t_ds) + [t_t]
    mean = Fraction(0)
    for i in range(m ** (N - 1)):
        tree = O.multi_tree(c, SEED, i, pattern=True)
        chain = O.multi_chain(c, SEED, i, pattern=True)
        assert (tree["dsi"], tree["settled"]) == (chain["dsi"], chain["settled"]), i
        w = Fraction(1)
        x = i
        for _ in range(N - 1):
            w *= pi[x % m]
            x //= m
        mean += w * tree["dsi"]
        assert tree["dsi"] <= N * t_t  # Thm 1 per trial
    assert mean == t_t + (N - 1) * sum(p * t for p, t in zip(pi, lat))


def test_thm1_per_trial_and_equality_at_zero_acceptance():
    rng = random.Random(13)
    for _ in range(40):
        m = rng.randint(2, 8)
        t_t = rng.randint(1, 50)
        t_ds = tuple(sorted(rng.randint(1, t_t) for _ in range(m - 1)))
        N = rng.randint(1, 60)
        rates = tuple(rng.random() for _ in range(m - 1))
        r = O.multi_run(O.MultiConfig(t_t, t_ds, rates, N), SEED, 0, 50)
        assert r["n_dsi_gt_nonsi"] == 0
        z = O.multi_run(O.MultiConfig(t_t, t_ds, (0.0,) * (m - 1), N), SEED, 0, 5)
        assert set(int(x) for x in z["dsi"]) == {N * t_t}
        one = O.multi_run(O.MultiConfig(t_t, t_ds, (1.0,) + rates[1:], N), SEED, 0, 5)
        assert set(int(x) for x in one["dsi"]) == {t_t + (N - 1) * t_ds[0]}


def test_appending_a_drafter_never_slows_a_trial():
    """Coupled per trial: drafters 1..m-1 keep their streams when drafter m (slower than all of
    them, no slower than the target) is appended; j* can only move to a faster model."""
    rng = random.Random(17)
    for _ in range(30):
        m = rng.randint(2, 7)
        t_t = rng.randint(2, 60)
        t_ds = tuple(sorted(rng.randint(1, t_t - 1) for _ in range(m - 1)))
        extra = rng.randint(t_ds[-1], t_t)
        rates = tuple(rng.random() for _ in range(m - 1))
        N = rng.randint(1, 50)
        base = O.multi_run(O.MultiConfig(t_t, t_ds, rates, N), SEED, 0, 30)
        more = O.multi_run(O.MultiConfig(t_t, t_ds + (extra,), rates + (rng.random(),), N), SEED, 0, 30)
        assert all(int(b) >= int(x) for b, x in zip(base["dsi"], more["dsi"]))


def test_monte_carlo_mean_within_six_sigma_of_exact_expectation():
    t_t, t_ds, N, T = 100, (5, 12, 30), 60, 4000
    rates = (0.55, 0.7, 0.85)
    c = O.MultiConfig(t_t, t_ds, rates, N)
    r = O.multi_run(c, SEED, 0, T, per_trial=False)
    thr = [Fraction(O.threshold(a), 1 << 32) for a in rates]
    pi, rest = [], Fraction(1)
    for a in thr:
        pi.append(rest * a)
        rest *= 1 - a
    pi.append(rest)
    lat = list(t_ds) + [t_t]
    e = t_t + (N - 1) * sum(p * t for p, t in zip(pi, lat))
    var = (N - 1) * (sum(p * t * t for p, t in zip(pi, lat)) - sum(p * t for p, t in zip(pi, lat)) ** 2)
    mean = Fraction(r["sum_dsi"], T)
    assert abs(float(mean - e)) <= 6 * float(var) ** 0.5 / T ** 0.5
    for j in range(4):
        f = r["sum_settled"][j] / (T * (N - 1))
        assert abs(f - float(pi[j])) <= 6 * (float(pi[j]) * (1 - float(pi[j])) / (T * (N - 1))) ** 0.5


def test_invalid_inputs_rejected():
    with pytest.raises(ValueError):
        O.multi_chain(O.MultiConfig(10, (5, 3), (0.5, 0.5), 4), SEED, 0)  # not ordered by latency
    with pytest.raises(ValueError):
        O.multi_chain(O.MultiConfig(10, (11,), (0.5,), 4), SEED, 0)  # drafter slower than target
    with pytest.raises(ValueError):
        O.multi_chain(O.MultiConfig(10, (1,), (1.5,), 4), SEED, 0)
    with pytest.raises(OverflowError):
        O.multi_tree(O.MultiConfig(100, (1, 2), (0.9, 0.9), 40), SEED, 0, max_threads=10000)


@pytest.mark.parametrize("N", [30, 60])
def test_tree_equals_chain_on_long_stream_trials(N):
    """The literal thread tree (every thread of Alg. 1) and the verified-chain
    simulation agree per trial at N = 30 and 60 on Philox-stream trials, for m = 2..5 and
    drafters slow enough (>= 0.2 t_m) for the tree to stay small."""
    rows = [(100, (25, 50), (0.5, 0.8)), (100, (20, 40, 60), (0.2, 0.5, 0.7)),
            (100, (30, 30, 50, 90), (0.5, 0.0, 0.4, 1.0)), (90, (45, 90), (0.95, 0.5)), (100, (50,), (0.1,))]
    for tt, tds, rates in rows:
        cfg = O.MultiConfig(tt, tds, rates, N, stream_id=N)
        for t in range(0, 2000, 13):
            lit = O.multi_tree(cfg, SEED, t, max_threads=1 << 20)
            ch = O.multi_chain(cfg, SEED, t)
            assert (lit["dsi"], lit["settled"]) == (ch["dsi"], ch["settled"]), (cfg, t)

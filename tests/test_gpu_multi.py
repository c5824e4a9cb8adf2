"""GPU parity of multi-drafter DSI (dsi_multi_simulate): Algorithm 1 with m
models, lookahead 1, through the C ABI against the CPU oracle
(oracle/dsi_oracle_multi.c).  Per-trial L_DSI and settled-by counts bit-exact, per-config
sums exact, FP64 means within 1e-9 relative; every outcome pattern of small N against the
literal thread-tree simulation; m = 2 against the single-drafter path at k = 1."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

D = pytest.importorskip("paper_2405_14105_b200.dsi_sim")
from paper_2405_14105_b200 import workloads as W  # noqa: E402

SEED = W.SEED


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def oracle_cfg(row, tick):
    nd = int(row["n_drafters"])
    return O.MultiConfig(O.ticks(float(row["t_target"]), tick),
                         tuple(O.ticks(float(x), tick) for x in row["t_drafter"][:nd]),
                         tuple(float(x) for x in row["accept_rate"][:nd]),
                         int(row["n_tokens"]), int(row["stream_id"]))


def offsets(cfgs):
    return np.concatenate([[0], np.cumsum(cfgs["n_trials"].astype(np.int64))])


def check(cfgs, tick, res, dsi, settled, pattern=False, tree=False):
    off = offsets(cfgs)
    for i, row in enumerate(cfgs):
        oc = oracle_cfg(row, tick)
        T = int(row["n_trials"])
        want = O.multi_run(oc, SEED, 0, T, pattern=pattern)
        m = oc.m
        got_d = dsi[off[i]:off[i + 1]].astype(np.int64)
        got_s = settled[off[i]:off[i + 1]]
        assert np.array_equal(got_d, want["dsi"]), (i, oc)
        assert np.array_equal(got_s[:, :m], want["settled"]), (i, oc)
        assert not got_s[:, m:].any()
        r = res[i]
        assert int(r["trials"]) == T and int(r["sum_dsi_ticks"]) == want["sum_dsi"]
        assert int(r["sumsq_dsi_ticks"]) == want["sumsq_dsi"]
        assert [int(x) for x in r["sum_settled"][:m]] == want["sum_settled"]
        assert int(r["n_dsi_gt_nonsi"]) == want["n_dsi_gt_nonsi"] == 0  # Thm 1
        assert int(r["nonsi_ticks"]) == want["nonsi"]
        mean = (float(want["sum_dsi"]) / float(T)) * tick
        assert abs(float(r["mean_dsi"]) - mean) <= 1e-9 * abs(mean)
        if tree:
            for t in range(T):
                lit = O.multi_tree(oc, SEED, t, pattern=pattern)
                assert int(got_d[t]) == lit["dsi"] and list(got_s[t, :m]) == lit["settled"], (i, t)


def tree_check(cfgs, tick, dsi, settled, per_cfg, budget=1 << 16, pattern=False):
    """Per-trial GPU results against the LITERAL thread tree of Alg. 1 (oracle_multi_tree, every
    thread spawned, terminated and relabelled as P:112-142 says), on up to per_cfg evenly spaced
    trials of each config; trials whose tree exceeds the thread budget are skipped.  Returns the
    number of trials checked (the chain simulation is never consulted here)."""
    off = offsets(cfgs)
    checked = 0
    for i, row in enumerate(cfgs):
        oc = oracle_cfg(row, tick)
        T = int(row["n_trials"])
        for t in np.unique(np.linspace(0, T - 1, min(per_cfg, T)).astype(int)):
            try:
                lit = O.multi_tree(oc, SEED, int(t), pattern=pattern, max_threads=budget)
            except OverflowError:
                continue
            assert int(dsi[off[i] + t]) == lit["dsi"], (i, int(t), oc)
            assert [int(x) for x in settled[off[i] + t, :oc.m]] == lit["settled"], (i, int(t), oc)
            checked += 1
    return checked


def test_fuzz_bit_exact_per_trial():
    cfgs, tick = W.multi_fuzz(60, n_max=70, trials=300)
    res, dsi, settled = D.dsi_multi_simulate(cfgs, tick=tick, seed=SEED, per_trial=True)
    check(cfgs, tick, res, dsi, settled)
    # the same trials against the literal thread tree wherever it fits a 65 536-thread budget
    assert tree_check(cfgs, tick, dsi, settled, per_cfg=40) >= 1500


# Latencies for which the literal thread tree stays small at N = 30..60 (drafters within ~4x of
# the target: the live tree is the set of model sequences whose summed latency fits in one
# target forward), m = 2..5, acceptance rates across [0, 1].
TREE_ROWS = [(1.0, (0.25, 0.5), (0.5, 0.8)), (1.0, (0.3, 0.6), (0.9, 0.9)),
             (1.0, (0.2, 0.4, 0.6), (0.2, 0.5, 0.7)), (1.0, (0.34,), (0.6,)),
             (1.0, (0.4, 0.7), (0.3, 0.6)), (1.0, (0.3, 0.3, 0.5, 0.9), (0.5, 0.0, 0.4, 1.0)),
             (0.9, (0.45, 0.9), (0.95, 0.5)), (1.0, (0.5,), (0.1,))]


@pytest.mark.parametrize("N", [30, 45, 60])
def test_literal_thread_tree_per_trial_at_n_30_to_60(N):
    """the multi-drafter kernel per trial against the literal thread tree
    (not the closed-form chain) at N = 30..60, 400 trials per config, ragged tile."""
    cfgs = W.multi_rows(TREE_ROWS, 1100, N, stream_id=N)
    res, dsi, settled = D.dsi_multi_simulate(cfgs, tick=0.01, seed=SEED, per_trial=True)
    assert tree_check(cfgs, 0.01, dsi, settled, per_cfg=400, budget=1 << 20) == 400 * len(TREE_ROWS)
    assert (res["n_dsi_gt_nonsi"] == 0).all()


def test_ragged_tiles_and_large_n():
    """Several 1024-trial tiles with a ragged tail; N > 4096 takes the per-call q half."""
    rows = [(1.0, (0.01, 0.05, 0.2), (0.6, 0.7, 0.9)), (1.0, (0.1,), (0.8,)),
            (1.0, (0.02, 0.02, 0.5, 0.5, 1.0, 1.0, 1.0), (0.3, 0.0, 0.5, 1.0, 0.2, 0.9, 0.4))]
    cfgs = W.multi_rows(rows, 2500, 101)
    big = W.multi_rows(rows[:2], 130, 5000, stream_id=7)
    for c in (cfgs, big):
        res, dsi, settled = D.dsi_multi_simulate(c, tick=0.01, seed=SEED, per_trial=True)
        check(c, 0.01, res, dsi, settled)


@pytest.mark.parametrize("t_t,t_ds,N", [(10, (2, 5), 7), (10, (4, 10), 6), (7, (1, 2, 3), 5),
                                        (9, (1, 4, 6, 9), 5), (12, (3,), 11)])
def test_every_pattern_against_the_literal_thread_tree(t_t, t_ds, N):
    m = len(t_ds) + 1
    rows = [(float(t_t), tuple(float(x) for x in t_ds), (0.5,) * (m - 1))]
    cfgs = W.multi_rows(rows, m ** (N - 1), N)
    res, dsi, settled = D.dsi_multi_simulate(cfgs, tick=1.0, seed=SEED, per_trial=True,
                                             flags=D.DSI_F_PATTERN)
    check(cfgs, 1.0, res, dsi, settled, pattern=True, tree=True)


def test_two_models_equal_single_drafter_path_at_k1():
    """m = 2, same seed and stream: the single-drafter kernel at k = 1 with SP >= ceil(t_t/t_d)
    (Prop. 1's setting) gives the same per-trial L_DSI and accept counts."""
    rows = [(1.0, (0.1,), (0.8,)), (1.0, (0.37,), (0.55,)), (0.5, (0.5,), (0.9,)), (1.0, (0.01,), (0.0,))]
    mc = W.multi_rows(rows, 3000, 100)
    res, dsi, settled = D.dsi_multi_simulate(mc, tick=0.01, seed=SEED, per_trial=True)
    sc = np.zeros(len(rows), W.CONFIG_DTYPE)
    for i, (tt, (td,), (a,)) in enumerate(rows):
        sc[i] = (tt, td, a, 1, int(np.ceil(round(tt / td, 9))), 100, 0, 3000, 0.0, 0.0)
    with D.Simulator(sc, tick=0.01, seed=SEED, flags=D.DSI_F_PER_TRIAL) as sim:
        sim.run()
        sres = sim.reduce()
        for i in range(len(rows)):
            tr = sim.trials(i)
            assert np.array_equal(tr["dsi"], dsi[i * 3000:(i + 1) * 3000]), i
            assert np.array_equal(tr["acc"], settled[i * 3000:(i + 1) * 3000, 0]), i
            assert int(sres[i]["sum_dsi_ticks"]) == int(res[i]["sum_dsi_ticks"])


def test_full_multi_heatmap_sampled_parity_and_exact_expectations():
    """The bench workload (10 100 configs x 1e4 trials, N = 100): the first 300 trials of 40
    evenly spaced configs bit-exact against the oracle (the trial index lives in the counter,
    so a shorter run is a prefix of the full one), and every config's Monte Carlo mean within
    6 sigma of its exact expectation t_m + (N-1) sum_j t_j pi_j."""
    cfgs, tick = W.multi_heatmap()
    res, _, _ = D.dsi_multi_simulate(cfgs, tick=tick, seed=SEED)
    assert (res["n_dsi_gt_nonsi"] == 0).all()
    assert (res["sum_settled"].sum(axis=1) == res["trials"].astype(np.int64) * 99).all()
    idx = np.linspace(0, len(cfgs) - 1, 40).astype(int)
    sub = cfgs[idx].copy()
    sub["n_trials"] = 300
    sres, sd, ss = D.dsi_multi_simulate(sub, tick=tick, seed=SEED, per_trial=True)
    check(sub, tick, sres, sd, ss)
    worst = 0.0
    for i, row in enumerate(cfgs):
        oc = oracle_cfg(row, tick)
        pi, rest = [], Fraction(1)
        for a in oc.accept_rates:
            p = Fraction(O.threshold(a), 1 << 32)
            pi.append(rest * p)
            rest *= 1 - p
        pi.append(rest)
        lat = list(oc.t_drafters) + [oc.t_target]
        e1 = sum(float(p) * t for p, t in zip(pi, lat))
        e2 = sum(float(p) * t * t for p, t in zip(pi, lat))
        n1 = oc.n_tokens - 1
        mean = oc.t_target + n1 * e1
        sd_ = (n1 * max(e2 - e1 * e1, 0.0)) ** 0.5
        T = int(row["n_trials"])
        got = int(res[i]["sum_dsi_ticks"]) / T
        if sd_ == 0:
            assert got == mean, i
        else:
            worst = max(worst, abs(got - mean) / (sd_ / T ** 0.5))
    assert worst < 6.0, worst


def test_invalid_configs_rejected_before_device_work():
    rows = [(1.0, (0.2, 0.1), (0.5, 0.5))]
    with pytest.raises(D.DsiError) as e:
        D.dsi_multi_simulate(W.multi_rows(rows, 10, 10), tick=0.01, seed=SEED)
    assert e.value.status == D.DSI_E_RANGE
    with pytest.raises(D.DsiError) as e:
        D.dsi_multi_simulate(W.multi_rows([(1.0, (0.005,), (0.5,))], 10, 10), tick=0.01, seed=SEED)
    assert e.value.status == D.DSI_E_TICK
    with pytest.raises(D.DsiError) as e:
        D.dsi_multi_simulate(W.multi_rows([(1e7, (1.0,), (0.5,))], 10, 1000), tick=0.01, seed=SEED)
    assert e.value.status == D.DSI_E_OVERFLOW


def test_max_n_and_single_token():
    """N = 32768 (the ABI's maximum) and N = 1 (no drafts: L = t_m)."""
    big = W.multi_rows([(1.0, (0.01, 0.1, 0.4), (0.3, 0.6, 0.9))], 40, 32768, stream_id=3)
    res, dsi, settled = D.dsi_multi_simulate(big, tick=0.01, seed=SEED, per_trial=True)
    check(big, 0.01, res, dsi, settled)
    one = W.multi_rows([(1.0, (0.1,), (0.5,)), (1.0, (0.1, 0.2), (0.9, 0.9))], 1000, 1)
    res, dsi, settled = D.dsi_multi_simulate(one, tick=0.01, seed=SEED, per_trial=True)
    assert (dsi == 100).all() and not settled.any()
    check(one, 0.01, res, dsi, settled)


@pytest.mark.parametrize("kw", [{"n_shards": 2}, {"n_shards": 7}, {"nccl": True}])
def test_partition_and_one_rank_nccl_bit_identical(kw):
    """The multi-GPU path on one device: the cost-balanced partition run as 2 or 7 shards back
    to back, and the NCCL all-reduce on a one-rank communicator, give the same integers."""
    cfgs, tick = W.multi_fuzz(40, seed=12, n_max=90, trials=5000)
    ref, _, _ = D.dsi_multi_simulate(cfgs, tick=tick, seed=SEED)
    if kw.get("nccl"):
        got, _, _ = D.dsi_multi_simulate(cfgs, tick=tick, seed=SEED, nccl_id=D.dsi_nccl_unique_id())
    else:
        got, _, _ = D.dsi_multi_simulate(cfgs, tick=tick, seed=SEED, **kw)
    for f in ("trials", "sum_dsi_ticks", "sumsq_dsi_ticks", "sum_settled", "n_dsi_gt_nonsi", "mean_dsi", "std_dsi"):
        assert np.array_equal(got[f], ref[f]), f


@pytest.mark.parametrize("name", ["heatmap", "fuzz"])
def test_means_only_shares_passes_across_latencies(name):
    """DSI_F_MEANS_ONLY: configs differing only in latencies share one kernel pass (j* depends on
    the indicators alone); sums, settled counts and means equal the default run bit for bit."""
    if name == "heatmap":
        cfgs, tick = W.multi_heatmap(trials=3000)
    else:
        base, tick = W.multi_fuzz(12, seed=21, n_max=80, trials=900)
        rows = []
        for b in base:  # each fuzz config again with every latency scaled: same indicator groups
            rows.append(b)
            c = b.copy()
            nd = int(c["n_drafters"])
            c["t_target"] = 2 * c["t_target"]
            c["t_drafter"][:nd] = c["t_drafter"][:nd] + 1
            rows.append(c)
        cfgs = np.array(rows, dtype=base.dtype)
    want, _, _ = D.dsi_multi_simulate(cfgs, tick=tick, seed=SEED)
    got, _, _ = D.dsi_multi_simulate(cfgs, tick=tick, seed=SEED, flags=D.DSI_F_MEANS_ONLY)
    for f in ("trials", "nonsi_ticks", "sum_dsi_ticks", "sum_settled", "n_dsi_gt_nonsi", "mean_dsi", "mean_nonsi"):
        assert np.array_equal(got[f], want[f]), f
    assert (got["sumsq_dsi_ticks"] == 0).all() and np.isnan(got["std_dsi"]).all()
    with pytest.raises(D.DsiError):
        D.dsi_multi_simulate(cfgs[:2], tick=tick, seed=SEED, flags=D.DSI_F_MEANS_ONLY, per_trial=True)


def test_golden_hand_traced_trees_on_the_gpu():
    """tests/golden/multi_drafter.json (hand-traced thread trees of Alg. 1, P:418's sum) from the
    GPU path in pattern mode (digit p-1 of the trial index in base m is j*(p) - 1)."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "multi_drafter.json")))["examples"]
    for e in g:
        m = len(e["t_drafters"]) + 1
        idx = sum((j - 1) * m ** p for p, j in enumerate(e["j_star"]))
        cfgs = W.multi_rows([(float(e["t_target"]), tuple(float(x) for x in e["t_drafters"]),
                              (0.5,) * (m - 1))], idx + 1, e["n_tokens"])
        res, dsi, settled = D.dsi_multi_simulate(cfgs, tick=1.0, seed=SEED, per_trial=True, flags=D.DSI_F_PATTERN)
        assert int(dsi[idx]) == e["dsi"], e["name"]
        assert [int(x) for x in settled[idx, :m]] == e["settled"], e["name"]
        assert int(res[0]["nonsi_ticks"]) == e["nonsi"]

"""GPU parity of the halves layout of the indicator stream (DSI_F_RNG_HALVES, R26).

Same bar as test_gpu_parity.py: per-trial records bit-exact against the oracle evaluating the
halves layout, integer sums exact, FP64 means within 1e-9.  The cases cover the tie path the
kernel takes with probability 2^-16 per position: thresholds whose T = thr >> 16 is an f16 NaN
pattern (the XOR form of the tie test), +-0 / +inf patterns (false-positive flags), T = 0 (every
acceptance a tie), T = 0xFFFF, thresholds built from the Philox outputs themselves so that given
positions tie, and enough trials that random ties occur.
"""
import numpy as np
import pytest

import oracle as O
from helpers import assert_result_equals_oracle, assert_trials_equal, oracle_sums

pytestmark = pytest.mark.gpu

D = pytest.importorskip("paper_2405_14105_b200.dsi_sim")
from paper_2405_14105_b200 import workloads as W  # noqa: E402

SEED = W.SEED
H = D.DSI_F_RNG_HALVES
ALL = D.DSI_F_PER_TRIAL | D.DSI_F_HIST


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_sim(cfgs, tick, flags, **kw):
    sim = D.Simulator(cfgs, tick=tick, seed=kw.pop("seed", SEED), flags=flags | H, **kw)
    sim.run()
    return sim, sim.reduce()


def check(sim, res, cfgs, tick, per_trial=True, hist=False, fresh=False, ctx="", idx=None):
    for i in (range(len(cfgs)) if idx is None else idx):
        want = oracle_sums(cfgs[i], tick, SEED, hist=hist, per_trial=per_trial, fresh=fresh, halves=True)
        assert_result_equals_oracle(res[i], want, tick, ctx=f"{ctx} cfg {i}")
        if per_trial:
            assert_trials_equal(sim.trials(i), want, ctx=f"{ctx} cfg {i}")
        if hist:
            seg, si = sim.hist(i)
            assert np.array_equal(seg, want["seg_hist"]), (ctx, i, "seg_hist")
            assert np.array_equal(si, want["si_hist"]), (ctx, i, "si_hist")


@pytest.mark.parametrize("flags", [ALL, D.DSI_F_PER_TRIAL])
def test_halves_fuzz_bit_exact(flags):
    cfgs, tick = W.fuzz(120, seed=31, trials=300)
    sim, res = run_sim(cfgs, tick, flags)
    check(sim, res, cfgs, tick, hist=bool(flags & D.DSI_F_HIST), ctx=f"fuzz {flags}")
    sim.close()


def test_halves_long_runs_and_pipelined_walk():
    """a in [0.85, 0.999], k up to 45 (k >= 30: the pipelined branch-free walk), N up to 300."""
    rng = np.random.default_rng(41)
    rows = []
    for i in range(60):
        t_t = int(rng.integers(2, 101))
        t_d = int(rng.integers(1, t_t + 1))
        k = int(rng.integers(30, 46)) if i % 2 else int(rng.integers(1, 30))
        rows.append((float(t_t), float(t_d), float(rng.uniform(0.85, 0.999)), k, int(rng.integers(1, 9)),
                     int(rng.integers(33, 301)), int(rng.integers(0, 3)), 200))
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 1.0, D.DSI_F_PER_TRIAL)
    check(sim, res, cfgs, 1.0, ctx="longruns")
    sim.close()


def test_halves_threshold_patterns():
    """T = thr >> 16 as an f16 bit pattern: NaN (0.49, 0.99: the XOR tie test), +inf
    (0x7C00), -0 (a = 0.5), +0 (a < 2^-16: every acceptance through a tie), 0xFFFF."""
    accs = [0.49, 0.99, 0.4844, 0x7C00 / 65536, 0.5, 2.0 ** -17, 3e-6, 1 - 2.0 ** -17, 0.8, 0.01]
    rows = [(1.0, 0.1, a, k, sp, n, s, 3000) for a in accs for (k, sp, n, s) in ((3, 4, 100, 0), (1, 7, 70, 1))]
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 0.01, D.DSI_F_PER_TRIAL)
    check(sim, res, cfgs, 0.01, ctx="thresholds")
    sim.close()


def _half(words, j):
    w = words[j % 4]
    return (w >> 16) if j < 4 else (w & 0xFFFF)


def test_halves_forced_ties():
    """Each config's threshold is built from the Philox outputs of one (trial, call) so that a
    chosen offset ties (v == T), with the tie-break deciding both ways; every call position in
    the 32-position word and a later word are covered."""
    key = (SEED & 0xFFFFFFFF, SEED >> 32)
    rows, N = [], 100
    for trial in (0, 3, 64):
        for q in (0, 1, 3, 6, 12):
            for j in range(8):
                v = _half(O.philox4x32_10((q, 0, trial, 0), key), j)
                w = _half(O.philox4x32_10((q, 1, trial, 0), key), j)
                for R in (w, min(w + 1, 0xFFFF)):
                    thr = (v << 16) | R
                    if 0 < thr:
                        rows.append((1.0, 0.2, thr / 2 ** 32, 2 + j % 5, 3, N, 0, 70))
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 0.01, D.DSI_F_PER_TRIAL)
    check(sim, res, cfgs, 0.01, ctx="forced ties")
    sim.close()


def test_halves_many_trials_random_ties():
    """2e5 trials x 99 positions: ~300 random ties on the kernel's rare path, per trial."""
    cfgs = W.rows([(1.0, 0.1, 0.8, 5, 2, 100, 0, 200_000), (1.0, 0.05, 0.37, 2, 7, 100, 2, 200_000)])
    sim, res = run_sim(cfgs, 0.01, D.DSI_F_PER_TRIAL)
    check(sim, res, cfgs, 0.01, ctx="many")
    sim.close()


def test_halves_long_sequences_and_arithmetic_path():
    """N = 1000 and N = 4097 (no shared-memory tables: per-call rounds 0-1, arithmetic costs)."""
    rows = [(1.0, 0.05, 0.9, 3, 7, 1000, 0, 257), (1.0, 0.3, 0.5, 2, 3, 4097, 1, 65),
            (1.0, 1.0, 0.97, 1, 1, 1000, 2, 130), (1.0, 0.3, 0.49, 40, 3, 4099, 0, 33)]
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 0.01, D.DSI_F_PER_TRIAL)
    check(sim, res, cfgs, 0.01, ctx="long")
    sim.close()


def test_halves_variants_ttft_fresh_k1():
    """The kernel's variants under the halves layout: TTFT configs, the fresh verifier
    (k t_d > t_t) and the k = 1 no-queue fast path (chosen when such configs carry the work)."""
    ttft = W.rows([(1.0, 0.1, 0.7, 4, 3, 80, 0, 500, 2.5, 0.3), (1.0, 0.2, 0.85, 2, 7, 64, 1, 500, 1.4, 0.2)])
    sim, res = run_sim(ttft, 0.01, D.DSI_F_PER_TRIAL)
    check(sim, res, ttft, 0.01, ctx="ttft")
    sim.close()
    fresh = W.rows([(1.0, 0.3, 0.9, 6, 3, 100, 0, 500), (1.0, 0.5, 0.6, 3, 2, 90, 1, 500)])
    sim, res = run_sim(fresh, 0.01, D.DSI_F_PER_TRIAL | D.DSI_F_FRESH_VERIFIER)
    check(sim, res, fresh, 0.01, fresh=True, ctx="fresh")
    sim.close()
    k1 = W.rows([(1.0, 0.2, a, 1, 7, 200, 0, 400) for a in (0.3, 0.6, 0.9, 0.99)])
    sim, res = run_sim(k1, 0.01, D.DSI_F_PER_TRIAL)
    check(sim, res, k1, 0.01, ctx="k1")
    sim.close()


def test_halves_bench_workload_sample():
    """cfg3 (the bench workload; every 40th heatmap cell, all k) in the bench's launch
    configuration (no test flags); 12 sampled configs against the oracle over all their trials."""
    cfgs, tick = W.cfg3(cells=slice(None, None, 40))
    sim, res = run_sim(cfgs, tick, 0)
    idx = np.random.default_rng(3).choice(len(cfgs), 12, replace=False)
    check(sim, res, cfgs, tick, per_trial=False, ctx="cfg3", idx=idx)
    # the law: mean acceptance within 6 sigma of a per config, pooled over the sample
    acc = res["sum_accepts"].astype(np.float64) / (cfgs["n_trials"] * 99.0)
    a = cfgs["accept_rate"]
    sd = np.sqrt(a * (1 - a) / (cfgs["n_trials"] * 99.0)) + 1e-12
    assert np.all(np.abs(acc - a) <= 6.5 * sd)
    sim.close()


MOMENTS = ("sum_dsi_ticks", "sum_si_ticks", "sumsq_dsi_ticks", "sumsq_si_ticks", "sum_segments",
           "sum_si_iters", "sum_accepts", "n_dsi_gt_nonsi", "n_dsi_gt_si", "trials")
MEANS = ("sum_dsi_ticks", "sum_si_ticks", "sum_segments", "sum_si_iters", "sum_accepts", "trials")


@pytest.mark.parametrize("name", ["cfg3_sample", "cfg4", "fuzz", "ttft_mix"])
@pytest.mark.parametrize("fresh", [False, True])
def test_halves_every_mode_bit_identical(name, fresh):
    """SHARED_STREAMS (fused and two-pass kernels) and MEANS_ONLY under the halves layout give the
    per-config kernel's integers (which the tests above pin to the oracle)."""
    if name == "cfg3_sample":
        cfgs, tick = W.cfg3(trials=2000, cells=slice(None, None, 11))
    elif name == "cfg4":
        cfgs, tick = W.cfg4(trials=3000)
    elif name == "fuzz":
        cfgs, tick = W.fuzz(150, seed=71, trials=500)
    else:
        cfgs = W.rows([(1.0, 0.1, 0.7, 4, 3, 80, 0, 500, 2.5, 0.3), (1.0, 0.2, 0.7, 2, 7, 80, 0, 500),
                       (1.0, 0.05, 0.49, 6, 5, 80, 1, 500, 1.5, 0.1), (1.0, 0.3, 0.49, 1, 7, 80, 1, 500)])
        tick = 0.01
        if fresh:
            pytest.skip("the fresh verifier excludes TTFT configs")
    base = D.DSI_F_FRESH_VERIFIER if fresh else 0
    _, want = run_sim(cfgs, tick, base)
    for mode, fields in ((D.DSI_F_SHARED_STREAMS, MOMENTS), (D.DSI_F_MEANS_ONLY, MEANS)):
        sim, got = run_sim(cfgs, tick, base | mode)
        for f in fields:
            assert np.array_equal(got[f], want[f]), (name, fresh, mode, f)
        sim.close()


def test_halves_bench_workload_full_size():
    """The bench workload (cfg3: 2.02 M configs x 1e4 trials, N 100) under the halves layout in the
    bench's launch configuration: sampled configs recomputed by the oracle over all their trials, the
    theorem counters on every config, and every one of the 2.02 M Monte Carlo means within 6 sigma of
    its exact expectation (the halves layout's law, Bernoulli(floor(a 2^32) / 2^32), at full scale)."""
    cfgs, tick = W.cfg3()
    sim, res = run_sim(cfgs, tick, D.DSI_F_TIMING)
    sim.close()
    assert np.all(res["trials"] == 10_000)
    idx = np.unique(np.concatenate([np.linspace(0, cfgs.size - 1, 16).round().astype(int),
                                    np.random.default_rng(5).integers(0, cfgs.size, 8)]))
    for i in idx:
        assert_result_equals_oracle(res[i], oracle_sums(cfgs[i], tick, SEED, halves=True), tick, ctx=f"cfg3[{i}]")
    kd = res["t_drafter_ticks"] * cfgs["lookahead"]
    inside = kd <= res["t_target_ticks"]
    assert np.all(res["n_dsi_gt_nonsi"][inside] == 0)
    assert np.all(res["n_dsi_gt_si"][inside & (res["eq1_feasible"] == 1)] == 0)
    from test_heatmap import exact_results
    ex = exact_results(cfgs, tick)
    for f, s in (("mean_si", "std_si"), ("mean_dsi", "std_dsi")):
        dev = np.abs(res[f] - ex[f])
        lim = 6.0 * res[s] / np.sqrt(10_000.0) + 1e-9 * ex[f]
        assert np.all(dev <= lim), (f, int(np.sum(dev > lim)))


def test_halves_large_monte_carlo_sampled():
    """BASELINE configs[4] (cfg5: 10 100 cells at the Eq.-1 lookahead, 1e5 trials, N 1000; mostly the
    k = 1 fast-path variant) under the halves layout; one config against the oracle over all its
    trials, the partition and Thm 1 on every config."""
    cfgs, tick = W.cfg5(D.dsi_min_lookahead)
    sim, res = run_sim(cfgs, tick, 0)
    sim.close()
    assert np.all(res["trials"] == cfgs["n_trials"])
    kd = res["t_drafter_ticks"] * cfgs["lookahead"]
    assert np.all(res["n_dsi_gt_nonsi"][kd <= res["t_target_ticks"]] == 0)
    i = 50 * 101 + 80  # t_d 0.51, a 0.80
    assert_result_equals_oracle(res[i], oracle_sums(cfgs[i], tick, SEED, halves=True), tick, ctx="cfg5")


@pytest.mark.parametrize("mode", [0, D.DSI_F_SHARED_STREAMS, D.DSI_F_MEANS_ONLY])
def test_halves_update_equals_a_fresh_handle(mode):
    """dsi_sim_update under the halves layout (device path where eligible): a handle updated to new
    config values gives the integers of a handle created with them."""
    a, tick = W.cfg3(trials=400, k_max=12, cells=slice(0, 404))  # 4 t_d x 101 a x k 1..12
    b = a.copy()  # new drafter latencies and lookaheads (as test_gpu_update_device.py)
    b["t_drafter"] = np.round(b["t_drafter"] * 2 + 0.01, 2)
    b["lookahead"] = np.maximum(1, 13 - b["lookahead"])
    sim = D.Simulator(a, tick=tick, seed=SEED, flags=mode | H)
    sim.run()
    sim.reduce()
    sim.update(b)
    got = sim.run().reduce()
    sim.close()
    _, want = run_sim(b, tick, mode)
    fields = MEANS if mode == D.DSI_F_MEANS_ONLY else MOMENTS
    for f in fields:
        assert np.array_equal(got[f], want[f]), (mode, f)


def _multi_oracle_cfg(row, tick):
    nd = int(row["n_drafters"])
    return O.MultiConfig(O.ticks(float(row["t_target"]), tick),
                         tuple(O.ticks(float(x), tick) for x in row["t_drafter"][:nd]),
                         tuple(float(x) for x in row["accept_rate"][:nd]),
                         int(row["n_tokens"]), int(row["stream_id"]), rng_halves=True)


@pytest.mark.parametrize("seed_fuzz", [17, 29])
def test_halves_multi_drafter_per_trial(seed_fuzz):
    """dsi_multi_simulate under the halves layout (drafter j on counter word 1 = 2(j-1), its
    tie-break on 2(j-1)+1): per-trial L_DSI and settled-by counts bit-exact against the oracle's
    chain, the literal thread tree on the small cases; thresholds with f16-NaN / zero high halves."""
    mf, mtick = W.multi_fuzz(40, seed=seed_fuzz, n_max=70, trials=120)
    rows = [(1.0, (0.02, 0.1), (0.49, 2.0 ** -17)), (1.0, (0.05, 0.2, 0.3), (0.99, 0.8, 0.5)),
            (1.0, (0.1,), (1 - 2.0 ** -17,))]
    extra = W.multi_rows(rows, 300, 90, stream_id=2)
    for cfgs, tick in ((mf, mtick), (extra, 0.01)):
        res, dsi, settled = D.dsi_multi_simulate(cfgs, tick=tick, seed=SEED, flags=H, per_trial=True)
        off = np.concatenate([[0], np.cumsum(cfgs["n_trials"].astype(np.int64))])
        for i, row in enumerate(cfgs):
            oc = _multi_oracle_cfg(row, tick)
            T = int(row["n_trials"])
            want = O.multi_run(oc, SEED, 0, T)
            got_d = dsi[off[i]:off[i + 1]].astype(np.int64)
            assert np.array_equal(got_d, want["dsi"]), (i, oc)
            assert np.array_equal(settled[off[i]:off[i + 1], :oc.m], want["settled"]), (i, oc)
            assert int(res[i]["sum_dsi_ticks"]) == want["sum_dsi"]
            if int(row["n_tokens"]) <= 9 and oc.m <= 4:
                for t in range(min(T, 20)):
                    assert int(got_d[t]) == O.multi_tree(oc, SEED, t)["dsi"], (i, t)


def test_halves_multi_drafter_one_drafter_is_the_single_drafter_stream():
    """m = 2 under the halves layout: the multi-drafter path at lookahead 1 equals the per-config
    path's halves stream (drafter 1 draws counter words 1 = 0 and 1, as the single-drafter layout)."""
    rows = [(1.0, (0.1,), (0.8,)), (1.0, (0.3,), (0.49,)), (1.0, (1.0,), (0.5,))]
    mc = W.multi_rows(rows, 500, 77)
    res, dsi, _ = D.dsi_multi_simulate(mc, tick=0.01, seed=SEED, flags=H, per_trial=True)
    single = W.rows([(1.0, r[1][0], r[2][0], 1, 100, 77, 0, 500) for r in rows])
    sim, sres = run_sim(single, 0.01, D.DSI_F_PER_TRIAL)
    for i in range(len(rows)):
        got = dsi[i * 500:(i + 1) * 500].astype(np.int64)
        assert np.array_equal(got, sim.trials(i)["dsi"].astype(np.int64)), i
    sim.close()

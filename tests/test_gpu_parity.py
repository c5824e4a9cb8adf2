"""GPU parity: the sm_100a path through the C ABI against the CPU oracle.

Per-trial records {acc, m, I, L_SI, L_DSI} must be bit-exact (integer ticks), the
per-config integer sums exact, and the FP64 means within 1e-9 relative (north_star).
Sizes span several tiles with ragged tails; the full-size bench workload is checked
on a sample of configs the oracle recomputes one by one, plus invariants.
"""
import math

import numpy as np
import pytest

import oracle as O
import exact_math as X
from helpers import assert_result_equals_oracle, assert_trials_equal, oracle_config, oracle_sums

pytestmark = pytest.mark.gpu

D = pytest.importorskip("paper_2405_14105_b200.dsi_sim")
from paper_2405_14105_b200 import workloads as W  # noqa: E402

SEED = W.SEED
ALL = D.DSI_F_PER_TRIAL | D.DSI_F_HIST


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_sim(cfgs, tick, flags=ALL, **kw):
    sim = D.Simulator(cfgs, tick=tick, seed=kw.pop("seed", SEED), flags=flags, **kw)
    sim.run()
    res = sim.reduce()
    return sim, res


def check_against_oracle(sim, res, cfgs, tick, per_trial=True, hist=True, pattern=False, ctx="",
                         fresh=False):
    for i, row in enumerate(cfgs):
        want = oracle_sums(row, tick, SEED, pattern=pattern, hist=hist, per_trial=per_trial, fresh=fresh)
        assert_result_equals_oracle(res[i], want, tick, ctx=f"{ctx} cfg {i}")
        if per_trial:
            assert_trials_equal(sim.trials(i), want, ctx=f"{ctx} cfg {i}")
        if hist:
            seg, si = sim.hist(i)
            assert np.array_equal(seg, want["seg_hist"]), (ctx, i, "seg_hist")
            assert np.array_equal(si, want["si_hist"]), (ctx, i, "si_hist")


def test_cfg1_bit_exact():
    cfgs, tick = W.cfg1(trials=1000)
    sim, res = run_sim(cfgs, tick)
    check_against_oracle(sim, res, cfgs, tick, ctx="cfg1")
    assert res[0]["eq1_feasible"] == 1 and res[0]["min_lookahead"] == 5
    sim.close()


def test_fuzz_bit_exact():
    """Edge cases: SP 1..8, k 1..12 and k > N, N in {1,2,3,..}, a in {0,1,rand}, Eq. 1 violated."""
    cfgs, tick = W.fuzz(160, seed=11, trials=300)
    sim, res = run_sim(cfgs, tick)
    check_against_oracle(sim, res, cfgs, tick, ctx="fuzz")
    sim.close()


def test_fuzz_long_runs_bit_exact():
    """Long runs of accepted drafts crossing 32-position words: a in [0.85, 0.999], N up to
    300, k in 1..40 (runs of >= k+1 ones inside a word, across words and at the end), SP 1..8."""
    rng = np.random.default_rng(21)
    rows = []
    for _ in range(60):
        t_t = int(rng.integers(2, 101))
        t_d = int(rng.integers(1, t_t + 1))
        rows.append((float(t_t), float(t_d), float(rng.uniform(0.85, 0.999)), int(rng.integers(1, 41)),
                     int(rng.integers(1, 9)), int(rng.integers(33, 301)), int(rng.integers(0, 3)), 200))
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 1.0)
    check_against_oracle(sim, res, cfgs, 1.0, ctx="longruns")
    sim.close()


def test_cfg2_table2_rows_subsample_bit_exact():
    cfgs, tick = W.cfg2(trials=2000)
    sim, res = run_sim(cfgs, tick)
    check_against_oracle(sim, res, cfgs, tick, ctx="cfg2")
    sim.close()


def test_cfg4_ragged_tiles_bit_exact():
    """N = 500 (16 Philox words), trials not a multiple of the block or the tile."""
    cfgs, tick = W.cfg4(trials=777)
    cfgs = cfgs[::9]
    sim, res = run_sim(cfgs, tick)
    check_against_oracle(sim, res, cfgs, tick, ctx="cfg4")
    sim.close()


def test_long_sequences_bit_exact():
    """N up to 1000 (config 5) and N = 4097 (an odd tail of the last Philox word)."""
    rows = [(1.0, 0.05, 0.9, 3, 7, 1000, 0, 257), (1.0, 0.3, 0.5, 2, 3, 4097, 1, 65),
            (1.0, 1.0, 0.97, 1, 1, 1000, 2, 130)]
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 0.01)
    check_against_oracle(sim, res, cfgs, 0.01, ctx="long")
    sim.close()


@pytest.mark.parametrize("N", [1, 2, 5, 12])
def test_pattern_mode_enumerates_every_pattern(N):
    """Enumeration mode: trial i's indicators are the bits of i; all 2^(N-1) patterns,
    each bit-exact against the oracle, and the weighted sum equals the exact h(g) form."""
    rows = [(100.0, 30.0, 0.5, 2, 2, N, 0, 1 << (N - 1)), (100.0, 7.0, 0.5, 4, 3, N, 0, 1 << (N - 1)),
            (100.0, 30.0, 0.5, 2, 1, N, 0, 1 << (N - 1))]
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 1.0, flags=ALL | D.DSI_F_PATTERN)
    check_against_oracle(sim, res, cfgs, 1.0, pattern=True, ctx=f"pattern N={N}")
    from fractions import Fraction
    for i, row in enumerate(cfgs):
        tr = sim.trials(i)
        a = Fraction(2, 3)

        def per_pattern(A):
            j = X.pattern_index(A)
            return {"dsi": int(tr["dsi"][j]), "iters": int(tr["iters"][j])}

        got = X.enumerate_expectations(N, a, per_pattern)
        want = X.expectations(N, int(row["lookahead"]), int(row["t_drafter"]), int(row["t_target"]),
                              int(row["sp_degree"]), a)
        assert got["dsi"] == want["dsi"] and got["iters"] == want["iters"]
    sim.close()


def test_shard_and_block_invariance():
    """The same seeded work split into 1..7 cost-balanced shards or run with other block
    sizes gives bit-identical per-trial records and sums (multi-GPU contract)."""
    cfgs, tick = W.fuzz(40, seed=3, trials=1000)
    base_sim, base = run_sim(cfgs, tick)
    base_tr = [base_sim.trials(i) for i in range(cfgs.size)]
    for kw in (dict(n_shards=2), dict(n_shards=3), dict(n_shards=7), dict(block_threads=32),
               dict(block_threads=64), dict(block_threads=96, n_shards=5)):
        sim, res = run_sim(cfgs, tick, **kw)
        for f in ("sum_dsi_ticks", "sum_si_ticks", "sumsq_dsi_ticks", "sum_segments", "n_dsi_gt_si"):
            assert np.array_equal(res[f], base[f]), (kw, f)
        for i in range(cfgs.size):
            assert_trials_equal(sim.trials(i), base_tr[i], ctx=str(kw))
        if kw.get("n_shards", 1) > 1:
            assert sim.launches() == kw["n_shards"] + 1  # + the reduce's partition check
        sim.close()
    base_sim.close()


def test_production_variant_matches_test_variant():
    """The kernel the bench runs (no per-trial records, no histograms) gives the same sums."""
    cfgs, tick = W.fuzz(60, seed=8, trials=900)
    sim_a, ra = run_sim(cfgs, tick, flags=ALL)
    sim_b, rb = run_sim(cfgs, tick, flags=0)
    for f in ("sum_dsi_ticks", "sum_si_ticks", "sumsq_dsi_ticks", "sumsq_si_ticks", "sum_segments",
              "sum_si_iters", "n_dsi_gt_nonsi", "n_dsi_gt_si", "mean_dsi", "std_dsi"):
        assert np.array_equal(ra[f], rb[f]), f
    sim_a.close()
    sim_b.close()


def ttft_fuzz(n, seed, trials):
    rng = np.random.default_rng(seed)
    base, _ = W.fuzz(n, seed=seed, trials=trials)
    for r in base:
        t_t, t_d = float(r["t_target"]), float(r["t_drafter"])
        t_t1 = float(rng.choice([t_t, rng.integers(1, 4 * t_t + 2), rng.integers(t_t, 12 * t_t + 2)]))
        t_d1 = float(rng.integers(1, int(min(t_t1, 5 * t_d + 3)) + 1))
        r["ttft_target"], r["ttft_drafter"] = t_t1, t_d1
    return base, 1.0


@pytest.mark.parametrize("flags", [0, ALL])
def test_ttft_fuzz_bit_exact(flags):
    """TTFT variant (N2): first forwards cost TTFT, incl. a first target forward much slower
    than later ones (threads finishing before thread 0) and TTFT below TPOT."""
    cfgs, tick = ttft_fuzz(150, seed=44, trials=250)
    sim, res = run_sim(cfgs, tick, flags=flags | D.DSI_F_PER_TRIAL)
    check_against_oracle(sim, res, cfgs, tick, hist=bool(flags & D.DSI_F_HIST), ctx=f"ttft {flags}")
    sim.close()


def test_ttft_table2_protocol_bit_exact():
    """Table 2's protocol with prefill: N = 50, SP 7, k in {1,5,10}, TTFT = Table-3
    ratio x TPOT, tick 0.001 ms."""
    cfgs, tick = W.cfg2_ttft(trials=1500)
    sim, res = run_sim(cfgs, tick, flags=0)
    check_against_oracle(sim, res, cfgs, tick, per_trial=False, hist=False, ctx="cfg2_ttft")
    sim.close()


def test_ttft_pattern_enumeration_exact():
    from fractions import Fraction
    N = 10
    rows = [(100.0, 14.0, 0.5, 1, 2, N, 0, 1 << (N - 1), 536.0, 15.0),
            (50.0, 7.0, 0.5, 2, 3, N, 0, 1 << (N - 1), 62.0, 9.0),
            (30.0, 10.0, 0.5, 3, 1, N, 0, 1 << (N - 1), 300.0, 12.0)]
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 1.0, flags=D.DSI_F_PATTERN | D.DSI_F_PER_TRIAL)
    check_against_oracle(sim, res, cfgs, 1.0, pattern=True, hist=False, ctx="ttft pattern")
    for i, row in enumerate(cfgs):
        tr = sim.trials(i)
        per = lambda A: {"dsi": int(tr["dsi"][X.pattern_index(A)]), "si": int(tr["si"][X.pattern_index(A)])}
        got = X.enumerate_expectations(N, Fraction(3, 4), per)
        want = X.expectations_ttft(N, int(row["lookahead"]), int(row["t_drafter"]), int(row["t_target"]),
                                   int(row["sp_degree"]), Fraction(3, 4), int(row["ttft_target"]),
                                   int(row["ttft_drafter"]))
        assert got["dsi"] == want["dsi"] and got["si"] == want["si"]
    sim.close()


MOMENTS = ("sum_dsi_ticks", "sum_si_ticks", "sumsq_dsi_ticks", "sumsq_si_ticks", "sum_segments",
           "sum_si_iters", "sum_accepts", "n_dsi_gt_nonsi", "n_dsi_gt_si", "trials", "mean_dsi", "std_dsi")


@pytest.mark.parametrize("fresh", [False, True], ids=["R1", "R24"])
@pytest.mark.parametrize("name", ["fuzz", "cfg2", "cfg3", "cfg4", "cfg5", "ragged"])
def test_shared_streams_bit_identical_to_default(name, fresh):
    """DSI_F_SHARED_STREAMS: one Philox pass per trial per group of configs
    with equal (stream, threshold, N, T); every per-config moment must equal the per-config
    mode's bit for bit (and so the oracle's, which that mode matches), under the literal
    reading (R1) and the fresh-verifier reading (R24) alike."""
    if name == "fuzz":
        cfgs, tick = W.fuzz(300, seed=31, trials=400)
    elif name == "cfg2":
        cfgs, tick = W.cfg2(trials=3000)
    elif name == "cfg3":
        cfgs, tick = W.cfg3(trials=1500, k_max=200, cells=slice(0, 10100, 37))
    elif name == "cfg4":
        cfgs, tick = W.cfg4(trials=2000)
    elif name == "cfg5":
        cfgs, tick = W.cfg5(D.dsi_min_lookahead, trials=300)
        cfgs = cfgs[::13]
    else:  # groups with trials not a multiple of the 128-trial tile, and a = 0 / a = 1 groups
        rows = [(1.0, 0.25, a, k, sp, 77, 0, 129 + 7 * k) for a in (0.0, 0.5, 1.0) for k in (1, 3, 9)
                for sp in (1, 7)]
        cfgs = W.rows(rows)
        tick = 0.01
    base_flags = FRESH if fresh else 0
    _, base = run_sim(cfgs, tick, flags=base_flags)
    sim, res = run_sim(cfgs, tick, flags=D.DSI_F_SHARED_STREAMS | base_flags)
    for f in MOMENTS:
        assert np.array_equal(res[f], base[f]), (name, fresh, f)
    if fresh and name in ("cfg3", "cfg4"):  # the variant acts on these (k t_d > t_t) ...
        _, lit = run_sim(cfgs, tick, flags=0)
        assert not np.array_equal(res["sum_dsi_ticks"], lit["sum_dsi_ticks"])
        assert (res["n_dsi_gt_nonsi"] == 0).all()  # ... and restores Thm 1
    sim.close()


@pytest.mark.parametrize("mix", ["ttft_only", "mixed", "mixed_big_groups"])
def test_shared_streams_with_ttft_configs(mix):
    """TTFT configs (first forwards, R23) in the shared-stream mode: they join no group and run
    through the per-config kernel's TTFT variant in the same dsi_sim_run, the other configs share
    their streams; every moment equals the per-config mode's, heatmap cells too, and an update
    that keeps which configs are TTFT works (one that changes it asks for a new handle)."""
    ttft, ttick = W.cfg2_ttft(trials=900)
    if mix == "ttft_only":
        cfgs, tick = ttft, ttick
    else:
        plain = ttft.copy()
        plain["ttft_target"] = 0.0
        plain["ttft_drafter"] = 0.0
        plain["stream_id"] = 1
        if mix == "mixed_big_groups":  # 256-thread two-pass plan for the shared part
            big, _ = W.cfg3(trials=900, k_max=12, cells=slice(0, 2525))
            big["t_target"] *= 10.0
            big["t_drafter"] *= 10.0  # (ticks of 0.001 ms: 0.1 ms steps)
            plain = np.concatenate([plain, big])
        cfgs = np.concatenate([ttft[::2], plain, ttft[1::2]])
        tick = ttick
    _, base = run_sim(cfgs, tick, flags=0)
    sim, res = run_sim(cfgs, tick, flags=D.DSI_F_SHARED_STREAMS)
    for f in MOMENTS:
        assert np.array_equal(res[f], base[f]), (mix, f)
    base_cells = D.dsi_heatmap(cfgs, base)
    cells = sim.run().heatmap()
    for f in cells.dtype.names:
        assert np.array_equal(cells[f], base_cells[f], equal_nan=cells[f].dtype.kind == "f"), (mix, f)
    new = cfgs.copy()
    # (a TTFT config is one whose first forwards differ from the later ones: R23)
    is_ttft = (((new["ttft_target"] != 0) & (np.abs(new["ttft_target"] - new["t_target"]) > 1e-9)) |
               ((new["ttft_drafter"] != 0) & (np.abs(new["ttft_drafter"] - new["t_drafter"]) > 1e-9)))
    new["t_target"] = new["t_target"] + 0.1 * is_ttft  # (the shared part's plan stays)
    sim.update(new)
    got = sim.run().reduce()
    _, want = run_sim(new, tick, flags=0)
    for f in MOMENTS:
        assert np.array_equal(got[f], want[f]), (mix, "update", f)
    flip = new.copy()
    i0 = int(np.nonzero(is_ttft)[0][0])
    flip["ttft_target"][i0] = 0.0  # config i0 stops being a TTFT config
    flip["ttft_drafter"][i0] = 0.0
    with pytest.raises(D.DsiError) as e:
        sim.update(flip)
    assert e.value.status == D.DSI_E_RANGE and "create a new handle" in str(e.value)
    sim.close()


@pytest.mark.parametrize("fresh", [False, True], ids=["R1", "R24"])
def test_shared_streams_against_oracle_sample(fresh):
    cfgs, tick = W.cfg3(trials=700, k_max=200, cells=slice(5, 10100, 1001))
    flags = D.DSI_F_SHARED_STREAMS | (FRESH if fresh else 0)
    sim, res = run_sim(cfgs, tick, flags=flags)
    for i in range(0, cfgs.size, 97):
        assert_result_equals_oracle(res[i], oracle_sums(cfgs[i], tick, SEED, fresh=fresh), tick, ctx=f"crn {i}")
    sim.close()


def test_shared_streams_options_are_validated():
    cfgs, tick = W.cfg1(trials=10)
    for bad in (D.DSI_F_PER_TRIAL, D.DSI_F_HIST, D.DSI_F_PATTERN):
        with pytest.raises(D.DsiError) as e:
            D.Simulator(cfgs, tick=tick, seed=SEED, flags=D.DSI_F_SHARED_STREAMS | bad)
        assert e.value.status == D.DSI_E_RANGE


@pytest.mark.parametrize("flags", [0, D.DSI_F_HIST, D.DSI_F_SHARED_STREAMS])
def test_nccl_one_rank_reduction_matches(flags):
    """The NCCL path of dsi_sim_reduce (dlopen'ed libnccl, ncclCommInitRank, ncclAllReduce
    of the u64 moments and histograms) on a one-rank communicator reproduces the local sums."""
    cfgs, tick = W.fuzz(30, seed=12, trials=500)
    _, base = run_sim(cfgs, tick, flags=flags)
    sim, res = run_sim(cfgs, tick, flags=flags, nccl_id=D.dsi_nccl_unique_id())
    for f in MOMENTS:
        assert np.array_equal(res[f], base[f]), f
    if flags & D.DSI_F_HIST:
        base_sim, _ = run_sim(cfgs, tick, flags=flags)
        for i in range(cfgs.size):
            a, b = sim.hist(i), base_sim.hist(i)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        base_sim.close()
    sim.close()


def test_seed_and_stream_change_the_draws():
    cfgs, tick = W.cfg1(trials=500)
    _, r1 = run_sim(cfgs, tick, flags=0)
    _, r2 = run_sim(cfgs, tick, flags=0, seed=SEED + 1)
    cfgs2 = cfgs.copy()
    cfgs2["stream_id"] = 9
    _, r3 = run_sim(cfgs2, tick, flags=0)
    assert r1["sum_dsi_ticks"][0] != r2["sum_dsi_ticks"][0]
    assert r1["sum_dsi_ticks"][0] != r3["sum_dsi_ticks"][0]


@pytest.mark.parametrize("name", ["cfg2", "cfg4", "cfg5"])
def test_other_baseline_configs_full_size_sampled(name):
    """BASELINE configs[1], [3], [4] at their full sizes (cfg2: Table-2 pairs x k {1,5,10}, 1e5
    trials, N 100; cfg4: k 1..20 x SP 2..8, 1e5 trials, N 500; cfg5: 10 100 cells at the Eq.-1
    lookahead, 1e5 trials, N 1000) in the per-config mode and in the shared-stream mode; sampled
    configs recomputed by the oracle over all their trials (exact sums), the partition and the
    theorem counters checked on every config."""
    if name == "cfg2":
        cfgs, tick = W.cfg2()
        pick = [0, 17, 29]
    elif name == "cfg4":
        cfgs, tick = W.cfg4()
        pick = [3, 131]
    else:
        cfgs, tick = W.cfg5(D.dsi_min_lookahead)
        pick = [50 * 101 + 80]  # t_d 0.51, a 0.80
    for flags in (0, D.DSI_F_SHARED_STREAMS):
        sim = D.Simulator(cfgs, tick=tick, seed=SEED, flags=flags)
        res = sim.run().reduce()
        sim.close()
        assert np.all(res["trials"] == cfgs["n_trials"])
        kd = res["t_drafter_ticks"] * cfgs["lookahead"]
        inside = kd <= res["t_target_ticks"]
        assert np.all(res["n_dsi_gt_nonsi"][inside] == 0)
        if flags == 0:
            base = res
            for i in pick:
                assert_result_equals_oracle(res[i], oracle_sums(cfgs[i], tick, SEED), tick, ctx=f"{name}[{i}]")
        else:
            for f in MOMENTS:
                assert np.array_equal(res[f], base[f]), (name, f)


def test_bench_workload_full_size_sampled():
    """The bench's workload (cfg3 heatmap, k <= 200, T = 1e4, N = 100) in the bench's launch
    configuration; a sample of configs is recomputed by the oracle one by one (exact sums),
    and properties that hold at any size are checked on all 2.02 M configs."""
    cfgs, tick = W.cfg3()
    sim = D.Simulator(cfgs, tick=tick, seed=SEED, flags=D.DSI_F_TIMING)
    sim.run()
    res = sim.reduce()
    assert np.all(res["trials"] == 10_000)
    idx = np.unique(np.linspace(0, cfgs.size - 1, 24).round().astype(int))
    rng = np.random.default_rng(1)
    idx = np.unique(np.concatenate([idx, rng.integers(0, cfgs.size, 8)]))
    for i in idx:
        want = oracle_sums(cfgs[i], tick, SEED)
        assert_result_equals_oracle(res[i], want, tick, ctx=f"cfg3[{i}]")
    # Thm 1 holds per trial wherever k t_d <= t_t; Thm 2 where also Eq. 1 holds (R6)
    kd = res["t_drafter_ticks"] * cfgs["lookahead"]
    inside = kd <= res["t_target_ticks"]
    assert np.all(res["n_dsi_gt_nonsi"][inside] == 0)
    assert np.all(res["n_dsi_gt_si"][inside & (res["eq1_feasible"] == 1)] == 0)
    # a = 0: DSI equals non-SI exactly (Thm 1 equality case); a = 1: one segment per trial
    a0 = cfgs["accept_rate"] == 0.0
    assert np.all(res["sum_dsi_ticks"][a0] == res["nonsi_ticks"][a0] * 10_000)
    a1 = cfgs["accept_rate"] == 1.0
    assert np.all(res["sum_segments"][a1] == 10_000)
    assert sim.kernel_ms() > 0
    sim.close()

    # every one of the 2.02 M Monte Carlo means sits within 6 sigma of its exact expectation
    from test_heatmap import exact_results
    ex = exact_results(cfgs, tick)
    T = 10_000.0
    for f, s in (("mean_si", "std_si"), ("mean_dsi", "std_dsi")):
        dev = np.abs(res[f] - ex[f])
        lim = 6.0 * res[s] / np.sqrt(T) + 1e-9 * ex[f]
        assert np.all(dev <= lim), (f, int(np.sum(dev > lim)))
    # the heatmap product of the GPU run against the exact one (Fig. 3 claims)
    cells = D.dsi_heatmap(cfgs, res)
    exact_cells = D.dsi_heatmap(cfgs, ex)
    assert cells.size == 10100
    assert np.all(cells["r_nonsi_dsi"] >= 1.0 - 1e-12)
    assert abs(cells["r_min_dsi"].max() - exact_cells["r_min_dsi"].max()) < 0.01
    clear = np.abs(cells["accept_rate"] - cells["t_drafter"]) > 0.05  # away from the a = t_d line
    assert np.array_equal((cells["r_nonsi_si"] > 1)[clear], (exact_cells["r_nonsi_si"] > 1)[clear])


def test_monte_carlo_mean_vs_exact_expectation():
    """Large-T GPU means sit within 6 sigma of the exact expectation (P11)."""
    from fractions import Fraction
    cfgs, tick = W.cfg1(trials=2_000_000)
    sim, res = run_sim(cfgs, tick, flags=0)
    r = res[0]
    p = Fraction(int(r["threshold"]), 2 ** 32)
    e = X.expectations(50, 5, 10, 100, 2, p)
    T = int(r["trials"])
    for mean, std, ex in ((r["mean_dsi"] / tick, r["std_dsi"] / tick, e["dsi"]),
                          (r["mean_si"] / tick, r["std_si"] / tick, e["si"])):
        assert abs(mean - float(ex)) < 6 * std / math.sqrt(T)
    sim.close()


def test_api_state_errors():
    cfgs, tick = W.cfg1(trials=10)
    sim = D.Simulator(cfgs, tick=tick, seed=SEED, flags=0)
    with pytest.raises(D.DsiError) as e:
        sim.reduce()
    assert e.value.status == D.DSI_E_STATE
    sim.run()
    with pytest.raises(D.DsiError) as e:
        sim.trials(0)
    assert e.value.status == D.DSI_E_STATE
    with pytest.raises(D.DsiError) as e:
        sim.hist(0)
    assert e.value.status == D.DSI_E_STATE
    with pytest.raises(D.DsiError) as e:
        sim.kernel_ms()
    assert e.value.status == D.DSI_E_STATE
    sim.reduce()
    sim.close()


def _changed(cfgs, dn=0, ttft=False):
    """Same trials per config; new acceptance, lookahead, N + dn (and TTFT).  a -> 1 - a and
    N -> N + dn are one-to-one, so the shared-stream grouping keeps its shape."""
    new = cfgs.copy()
    new["accept_rate"] = 1.0 - cfgs["accept_rate"]
    new["lookahead"] = cfgs["lookahead"] % 7 + 1
    new["n_tokens"] = cfgs["n_tokens"] + dn
    if ttft:
        new["ttft_target"] = new["t_target"] * 3
        new["ttft_drafter"] = new["t_drafter"] * 2
    return new


@pytest.mark.parametrize("flags,dn,ttft", [(0, 300, True), (ALL, 30, True), (0, 5000, False),
                                           (D.DSI_F_SHARED_STREAMS, 900, False)])
def test_update_matches_a_fresh_handle(flags, dn, ttft):
    """dsi_sim_update may grow N past the create-time maximum (shared-memory tables are
    sized per launch) and switch the TTFT variant on; results equal a fresh handle's."""
    cfgs, tick = W.fuzz(40, seed=77, trials=300)
    if flags & D.DSI_F_HIST:  # HIST fixes min(k, N) per config
        cfgs["lookahead"] = cfgs["lookahead"] % 7 + 1
        cfgs["n_tokens"] = np.maximum(cfgs["n_tokens"], 8)
    new = _changed(cfgs, dn, ttft)
    if flags & D.DSI_F_HIST:
        new["lookahead"] = cfgs["lookahead"]
    sim, _ = run_sim(cfgs, tick, flags=flags)
    sim.update(new).run()
    got = sim.reduce()
    _, want = run_sim(new, tick, flags=flags)
    for f in MOMENTS:
        assert np.array_equal(got[f], want[f]), f
    if flags & D.DSI_F_PER_TRIAL:
        for i in range(0, new.size, 9):
            assert_result_equals_oracle(got[i], oracle_sums(new[i], tick, SEED), tick, ctx=f"upd {i}")
    sim.close()


def test_update_growing_n_in_the_two_pass_shared_stream_form():
    """the two-pass shared-stream form (groups of >= 256 configs: here 101
    acceptance groups of 400 (t_d, k) configs) keeps per-trial run records whose size grows
    with N; an update from N = 100 to 120 keeps the record count but not the bytes, and must
    equal a fresh handle (the buffer is re-sized by bytes, not records)."""
    cfgs, tick = W.cfg3(trials=512, k_max=20, cells=slice(0, 2020))
    new = cfgs.copy()
    new["n_tokens"] = 120  # (keeps 256-thread blocks: the group and unit counts stay)
    flags = D.DSI_F_SHARED_STREAMS
    sim, _ = run_sim(cfgs, tick, flags=flags)
    sim.update(new).run()
    got = sim.reduce()
    _, want = run_sim(new, tick, flags=flags)
    _, plain = run_sim(new, tick, flags=0)
    for f in MOMENTS:
        assert np.array_equal(got[f], want[f]), f
        assert np.array_equal(got[f], plain[f]), f
    sim.close()


def test_failed_update_keeps_previous_configs():
    cfgs, tick = W.fuzz(20, seed=3, trials=200)
    sim, before = run_sim(cfgs, tick, flags=0)
    bad = cfgs.copy()
    bad["accept_rate"][4] = 1.5
    with pytest.raises(D.DsiError) as e:
        sim.update(bad)
    assert e.value.status == D.DSI_E_RANGE
    after = sim.run().reduce()
    for f in MOMENTS:
        assert np.array_equal(after[f], before[f]), f
    sim.close()
    # shared streams: an update that changes the grouping is refused, the plan kept
    sim, before = run_sim(cfgs, tick, flags=D.DSI_F_SHARED_STREAMS)
    regroup = cfgs.copy()
    regroup["stream_id"], regroup["accept_rate"], regroup["n_tokens"] = 0, 0.5, 50  # one group
    with pytest.raises(D.DsiError) as e:
        sim.update(regroup)
    assert e.value.status == D.DSI_E_RANGE
    after = sim.run().reduce()
    for f in MOMENTS:
        assert np.array_equal(after[f], before[f]), f
    # growing N past the shared-stream limit is refused too
    big = cfgs.copy()
    big["n_tokens"] = 2049
    with pytest.raises(D.DsiError) as e:
        sim.update(big)
    assert e.value.status == D.DSI_E_RANGE
    sim.close()


def test_shared_streams_at_max_n():
    """N = 2048 (the shared-stream limit: 128 run lists of N/3 + 2 entries in shared memory)."""
    rows = [(1.0, td, a, k, 7, 2048, 0, 256) for td in (0.05, 0.5) for a in (0.5, 0.9, 0.99)
            for k in (1, 4, 30)]
    cfgs, tick = W.rows(rows), 0.01
    _, base = run_sim(cfgs, tick, flags=0)
    sim, res = run_sim(cfgs, tick, flags=D.DSI_F_SHARED_STREAMS)
    for f in MOMENTS:
        assert np.array_equal(res[f], base[f]), f
    sim.close()


FRESH = D.DSI_F_FRESH_VERIFIER


@pytest.mark.parametrize("flags", [0, ALL])
def test_fresh_verifier_fuzz_bit_exact(flags):
    """the fresh-verifier variant through the C ABI against
    the oracle's event simulation, per trial (flags ALL) and in the production walk."""
    cfgs, tick = W.fuzz(160, seed=41, trials=192)
    assert np.sum(cfgs["lookahead"] * cfgs["t_drafter"] > cfgs["t_target"]) > 40
    sim, res = run_sim(cfgs, tick, flags=flags | FRESH)
    check_against_oracle(sim, res, cfgs, tick, per_trial=bool(flags), hist=bool(flags), ctx="fresh",
                         fresh=True)
    assert np.all(res["n_dsi_gt_nonsi"] == 0)  # Thm 1 per trial
    sim.close()


def test_fresh_verifier_pattern_enumeration():
    """Every pattern of N <= 12 against the hand-derived closed form (exact_math.C_fresh)."""
    rows = [(10.0, 4.0, 0.5, 5, 1, 12, 0, 1 << 11), (100.0, 14.0, 0.5, 20, 7, 12, 0, 1 << 11),
            (40.0, 30.0, 0.5, 3, 2, 11, 0, 1 << 10), (12.0, 11.0, 0.5, 2, 3, 10, 0, 1 << 9),
            (9.0, 2.0, 0.5, 7, 1, 12, 0, 1 << 11)]
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 1.0, flags=D.DSI_F_PATTERN | D.DSI_F_PER_TRIAL | FRESH)
    for i, r in enumerate(rows):
        t_t, t_d, _, k, sp, N, _, T = r
        got = sim.trials(i)
        for idx in range(T):
            A = [(idx >> p) & 1 for p in range(N - 1)]
            want = X.closed_form_fresh(A, N, k, int(t_d), int(t_t), sp)
            assert int(got["dsi"][idx]) == want["dsi"], (r, A)
            assert int(got["si"][idx]) == want["si"], (r, A)
    sim.close()


def test_fresh_verifier_cfg4_sweep():
    """Config 4 (k = 1..20 x SP 2..8, t_d = t_t/10): k > 10 is where the variant acts."""
    cfgs, tick = W.cfg4(trials=3000)
    _, base = run_sim(cfgs, tick, flags=0)
    sim, res = run_sim(cfgs, tick, flags=FRESH)
    act = cfgs["lookahead"] * cfgs["t_drafter"] > cfgs["t_target"] + 1e-12
    for f in MOMENTS:
        assert np.array_equal(res[f][~act], base[f][~act]), f
    assert np.all(res["sum_dsi_ticks"][act] < base["sum_dsi_ticks"][act])
    assert np.all(res["n_dsi_gt_nonsi"] == 0)
    for i in np.nonzero(act)[0][::9]:
        want = oracle_sums(cfgs[i], tick, SEED, count=3000, fresh=True)
        assert_result_equals_oracle(res[i], want, tick, ctx=f"cfg4 fresh {i}")
    sim.close()


def test_fresh_verifier_long_sequences_arithmetic_path():
    """N > 4096 (no shared-memory tables: segment costs by arithmetic)."""
    cfgs = W.rows([(100.0, 30.0, a, k, sp, 5000, 0, 64) for a, k, sp in
                   ((0.9, 7, 1), (0.99, 40, 3), (0.5, 4, 2))])
    sim, res = run_sim(cfgs, 1.0, flags=FRESH | D.DSI_F_PER_TRIAL)
    check_against_oracle(sim, res, cfgs, 1.0, hist=False, ctx="fresh N5000", fresh=True)
    sim.close()


def test_fresh_verifier_options():
    """The fresh-verifier reading is accepted in every mode (round 2) but not with TTFT configs."""
    cfgs, tick = W.cfg1(trials=10)
    for extra in (0, D.DSI_F_SHARED_STREAMS, D.DSI_F_MEANS_ONLY):
        D.Simulator(cfgs, tick=tick, seed=SEED, flags=FRESH | extra).close()
    ttft, ttick = W.cfg2_ttft(trials=10)
    for extra in (0, D.DSI_F_SHARED_STREAMS):
        with pytest.raises(D.DsiError) as e:
            D.Simulator(ttft, tick=ttick, seed=SEED, flags=FRESH | extra)
        assert e.value.status == D.DSI_E_RANGE


def _assert_cells_equal(got, want, ctx=""):
    assert got.size == want.size, ctx
    for f in want.dtype.names:
        np.testing.assert_array_equal(got[f], want[f], err_msg=f"{ctx} {f}")


@pytest.mark.parametrize("mode", ["default", "shared", "fresh", "ttft", "nccl"])
def test_device_heatmap_equals_host_heatmap(mode):
    """dsi_sim_heatmap (argmin over k on the device) == dsi_heatmap over
    dsi_sim_reduce's results, every field bit for bit (NaN where no k satisfies Eq. 1)."""
    flags, kw = 0, {}
    if mode == "ttft":
        cfgs, tick = W.cfg2_ttft(trials=2000)
    elif mode == "default":  # k <= 10: the t_d = 0.01 cells have no Eq.-1-feasible k (need k >= 15)
        cfgs, tick = W.cfg3(trials=400, k_max=10, cells=slice(0, 10100, 29))
    else:
        cfgs, tick = W.cfg3(trials=400, k_max=200, cells=slice(3, 10100, 53))
    if mode == "shared":
        flags = D.DSI_F_SHARED_STREAMS
    elif mode == "fresh":
        flags = FRESH
    elif mode == "nccl":
        kw["nccl_id"] = D.dsi_nccl_unique_id()
    sim, res = run_sim(cfgs, tick, flags=flags, **kw)
    want = D.dsi_heatmap(cfgs, res)
    got = sim.heatmap()
    _assert_cells_equal(got, want, mode)
    assert np.any(got["dsi_lookahead"] == -1) == (mode == "default")
    assert np.isnan(got["dsi"]).sum() == np.sum(got["dsi_lookahead"] == -1)
    sim.close()


def test_device_heatmap_after_update_and_state():
    cfgs, tick = W.cfg3(trials=200, k_max=20, cells=slice(0, 10100, 97))
    sim = D.Simulator(cfgs, tick=tick, seed=SEED)
    n = ctypes_count(sim)
    assert n == cfgs.size // 20
    with pytest.raises(D.DsiError) as e:
        sim.heatmap()
    assert e.value.status == D.DSI_E_STATE
    new = cfgs.copy()
    new["accept_rate"] = np.round(1.0 - cfgs["accept_rate"], 2)
    sim.update(new).run()
    got = sim.heatmap()
    _, res = run_sim(new, tick, flags=0)
    _assert_cells_equal(got, D.dsi_heatmap(new, res), "update")
    sim.close()


def ctypes_count(sim):
    import ctypes
    n = ctypes.c_size_t()
    assert D.lib.dsi_sim_heatmap(sim.h, None, 0, ctypes.byref(n)) == 0
    return n.value


def test_shared_streams_update_with_same_keys_keeps_plan():
    """An update that keeps every plan key (stream, threshold, N, T, k, t_t, t_d, SP) reuses
    the shared-stream plan; results equal a fresh handle's, also after a re-planning update."""
    cfgs, tick = W.cfg3(trials=300, k_max=30, cells=slice(0, 10100, 211))
    sim, first = run_sim(cfgs, tick, flags=D.DSI_F_SHARED_STREAMS)
    sim.update(cfgs.copy()).run()
    again = sim.reduce()
    for f in MOMENTS:
        assert np.array_equal(again[f], first[f]), f
    new = cfgs.copy()
    new["lookahead"] = 31 - cfgs["lookahead"]  # same grouping, new order inside groups
    sim.update(new).run()
    got = sim.reduce()
    _, want = run_sim(new, tick, flags=D.DSI_F_SHARED_STREAMS)
    for f in MOMENTS:
        assert np.array_equal(got[f], want[f]), f
    sim.close()


@pytest.mark.parametrize("kw", [dict(), dict(n_shards=3), dict(n_shards=7)])
def test_two_pass_shared_streams_ragged_and_sharded(kw):
    """The two-pass shared-stream form (groups >= 256 configs: pass 1 writes each trial's
    record once, pass 2 streams tile records with bulk copies) with trial counts that are not
    multiples of the 256-trial tile and several shards per device (each shard's pass-1 tile
    list): bit-identical to the default mode."""
    cfgs, tick = W.cfg3(trials=1000, k_max=40)
    a100 = np.rint(cfgs["accept_rate"] * 100).astype(np.int64)
    cfgs = cfgs[np.isin(a100, [0, 45, 70, 93, 100])].copy()  # 5 groups of 4000 configs (t_d x k)
    a100 = np.rint(cfgs["accept_rate"] * 100).astype(np.int64)
    cfgs["n_trials"] = 700 + 13 * (a100 % 7)  # ragged: not multiples of the 256-trial tile
    _, base = run_sim(cfgs, tick, flags=0)
    sim, res = run_sim(cfgs, tick, flags=D.DSI_F_SHARED_STREAMS, **kw)
    for f in MOMENTS:
        assert np.array_equal(res[f], base[f]), (kw, f)
    sim.close()


def test_max_n_bit_exact():
    """N = 32768, the largest the ABI accepts (arithmetic segment costs, 8192 Philox calls per
    trial), with and without queueing, and the fresh-verifier variant (k t_d > t_t)."""
    rows = [(1.0, 0.1, 0.9, 4, 3, 32768, 0, 40), (1.0, 0.5, 0.6, 1, 1, 32768, 5, 33)]
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 0.01, flags=D.DSI_F_PER_TRIAL)
    check_against_oracle(sim, res, cfgs, 0.01, hist=False, ctx="maxN")
    sim.close()
    fr = W.rows([(1.0, 0.5, 0.7, 3, 2, 32768, 1, 20)])
    sim, res = run_sim(fr, 0.01, flags=D.DSI_F_PER_TRIAL | D.DSI_F_FRESH_VERIFIER)
    check_against_oracle(sim, res, fr, 0.01, hist=False, fresh=True, ctx="maxN fresh")
    sim.close()


def test_max_trials_every_trial_counted_once():
    """n_trials = 2^32, the largest the ABI accepts (the 32-bit trial counter word takes every
    value): the on-device partition check passes, N = 1 sums are exact (L = t_t, no draws), and
    at N = 2 the one indicator per trial is Binomial(2^32, thr/2^32) within 6 sigma with L_DSI,
    L_SI determined by it (A_1 = 1: one segment of 2; A_1 = 0: two of 1)."""
    T = 1 << 32
    cfgs = W.rows([(1.0, 0.2, 0.7, 3, 2, 1, 0, T), (1.0, 0.2, 0.7, 3, 2, 2, 0, T)])
    sim, res = run_sim(cfgs, 0.01, flags=0)
    r1, r2 = res[0], res[1]
    assert int(r1["trials"]) == T and int(r1["sum_dsi_ticks"]) == 100 * T and int(r1["sum_si_ticks"]) == 160 * T
    assert int(r1["sum_accepts"]) == 0 and int(r1["sum_segments"]) == T
    acc = int(r2["sum_accepts"])
    p = int(r2["threshold"]) / 2 ** 32
    assert abs(acc - T * p) <= 6 * math.sqrt(T * p * (1 - p))
    # g = 2 costs t_t + S(1) = 100 + 60; two segments of 1 cost 2 t_t; SI: 1 iteration (k+1 >= 2)
    # for A_1 = 1, 2 iterations for A_1 = 0, each k t_d + t_t = 160
    assert int(r2["sum_dsi_ticks"]) == acc * 160 + (T - acc) * 200
    assert int(r2["sum_si_ticks"]) == acc * 160 + (T - acc) * 320
    assert int(r2["trials"]) == T
    sim.close()


def test_reduce_to_root_flag_on_rank_zero():
    """DSI_F_REDUCE_TO_ROOT: rank 0 (here the only rank, through a one-rank NCCL communicator)
    gets exactly the results of the default reduce."""
    cfgs, tick = W.fuzz(40, seed=8, trials=500)
    _, want = run_sim(cfgs, tick, flags=0)
    sim, got = run_sim(cfgs, tick, flags=D.DSI_F_REDUCE_TO_ROOT, nccl_id=D.dsi_nccl_unique_id())
    for f in want.dtype.names:
        assert np.array_equal(got[f], want[f]) or np.allclose(got[f], want[f], equal_nan=True), f
    sim.close()


@pytest.mark.parametrize("case", ["worst_case", "best_case"])
def test_table1_on_the_gpu(case):
    """Table 1 straight from the GPU path: tokens generated by t1..t4 with a 14%
    drafter, lookahead 1, SP 7 (tests/golden/table1.json), from one trial per N = 1..79."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")))
    a = g[case]["accept_rate"]
    rows = [(float(g["t_target"]), float(g["t_drafter"]), a, g["lookahead"], g["sp_degree"], n, 0, 1)
            for n in range(1, 80)]
    sim, res = run_sim(W.rows(rows), 1.0, flags=0)
    lat = {"nonsi": res["nonsi_ticks"], "si": res["sum_si_ticks"], "dsi": res["sum_dsi_ticks"]}
    for alg in ("nonsi", "si", "dsi"):
        counts = [max(n for n in range(1, 80) if lat[alg][n - 1] <= t) for t in g["times"]]
        assert counts == g[case][alg], (case, alg, counts)
    sim.close()


def test_worked_examples_on_the_gpu():
    """The hand-derived examples of tests/golden/worked_examples.json (Prop. 1's 426, the SP=2 / SP=1
    schedules 540 / 700, S:202's 1020 ms, ...) straight from the GPU path: pattern mode reads
    the example's acceptance pattern from the trial index (A_p = bit p-1), a = 0 / 1 otherwise."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))["examples"]
    for e in g:
        N = e["n_tokens"]
        A = e["A"]
        if isinstance(A, list):
            idx = sum(bit << p for p, bit in enumerate(A))
            row = [(float(e["t_target"]), float(e["t_drafter"]), 0.5, e["lookahead"], e["sp_degree"], N, 0, idx + 1)]
            sim, res = run_sim(W.rows(row), 1.0, flags=D.DSI_F_PATTERN | D.DSI_F_PER_TRIAL)
            tr = sim.trials(0, idx, 1)
            got = {"dsi": int(tr["dsi"][0]), "si": int(tr["si"][0]), "iters": int(tr["iters"][0])}
        else:
            a = 1.0 if A == "all1" else 0.0
            row = [(float(e["t_target"]), float(e["t_drafter"]), a, e["lookahead"], e["sp_degree"], N, 0, 1)]
            sim, res = run_sim(W.rows(row), 1.0, flags=D.DSI_F_PER_TRIAL)
            tr = sim.trials(0)
            got = {"dsi": int(tr["dsi"][0]), "si": int(tr["si"][0]), "iters": int(tr["iters"][0])}
        got["nonsi"] = int(res[0]["nonsi_ticks"])
        for key in ("dsi", "si", "iters", "nonsi"):
            if key in e:
                assert got[key] == e[key], (e["name"], key, got[key])
        sim.close()


def test_fresh_verifier_golden_on_the_gpu():
    """tests/golden/fresh_verifier.json (hand-derived schedules of R24) from the GPU path, with and
    without DSI_F_FRESH_VERIFIER."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fresh_verifier.json")))["examples"]
    e = g[0]
    rows = [(float(e["t_target"]), float(e["t_drafter"]), 1.0, e["lookahead"], e["sp_degree"], n, 0, 1)
            for n in range(1, len(e["dsi_by_n_tokens"]) + 1)]
    for flags, want in ((FRESH, e["dsi_by_n_tokens"]), (0, e["default_dsi_by_n_tokens"])):
        sim, res = run_sim(W.rows(rows), 1.0, flags=flags)
        assert [int(x) for x in res["sum_dsi_ticks"]] == want, flags
        sim.close()
    e = g[1]
    idx = sum(bit << p for p, bit in enumerate(e["A"]))
    row = [(float(e["t_target"]), float(e["t_drafter"]), 0.5, e["lookahead"], e["sp_degree"], e["n_tokens"], 0,
            idx + 1)]
    for flags, key in ((FRESH, "dsi"), (0, "default_dsi")):
        sim, _ = run_sim(W.rows(row), 1.0, flags=flags | D.DSI_F_PATTERN | D.DSI_F_PER_TRIAL)
        tr = sim.trials(0, idx, 1)
        assert int(tr["dsi"][0]) == e[key], key
        if key == "dsi":
            assert int(tr["si"][0]) == e["si"]
        sim.close()


@pytest.fixture
def k1_fast_forced():
    """The test build with the planner's k1_fast knob on (include/dsi_sim_testing.h); its kernels
    are compiled from the same sources as the product's."""
    with D.use_library("test"):
        D.dsi_test_set_knob("k1_fast", 1)
        try:
            yield
        finally:
            D.dsi_test_set_knob("k1_fast", -1)


def test_k1_fast_path_fuzz_bit_exact(k1_fast_forced):
    """The k = 1 no-queue fast path (parity of segment ends instead of the run walk, VAR 3), forced
    on for the fuzz set: every trial bit-exact against the oracle."""
    cfgs, tick = W.fuzz(160, seed=11, trials=300)
    sim, res = run_sim(cfgs, tick, flags=D.DSI_F_PER_TRIAL)
    check_against_oracle(sim, res, cfgs, tick, hist=False, ctx="k1fast")
    sim.close()


@pytest.mark.parametrize("N", [2, 5, 12, 33])
def test_k1_fast_path_every_pattern(k1_fast_forced, N):
    rows = [(1.0, 0.2, 0.5, 1, 7, N, 0, min(1 << (N - 1), 1 << 16)), (1.0, 1.0, 0.5, 1, 1, N, 0, min(1 << (N - 1), 1 << 16))]
    cfgs = W.rows(rows)
    sim, res = run_sim(cfgs, 0.01, flags=D.DSI_F_PER_TRIAL | D.DSI_F_PATTERN)
    check_against_oracle(sim, res, cfgs, 0.01, hist=False, pattern=True, ctx=f"k1fast N={N}")
    sim.close()


def test_cfg5_subsample_bit_exact():
    """Config 5 (k = Eq.-1 minimum at SP 7: mostly k = 1 without queueing, so the fast-path variant
    is chosen automatically), N = 1000: every trial of a 50-config sample bit-exact."""
    cfgs, tick = W.cfg5(D.dsi_min_lookahead, trials=200)
    cfgs = cfgs[::202].copy()
    sim, res = run_sim(cfgs, tick, flags=D.DSI_F_PER_TRIAL)
    check_against_oracle(sim, res, cfgs, tick, hist=False, ctx="cfg5")
    sim.close()

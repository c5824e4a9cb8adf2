"""GPU tests of the means-only mode (DSI_F_MEANS_ONLY, SURVEY 8(f) N3 "aggregate H[g]").

Per group of configs that draw identical indicators, one pass builds the segment-length
histogram H[g]; every config's sums follow by linearity over segments.  Those are the same
integers the per-trial kernels add, so every sum (and hence every mean and every heatmap
cell) must be bit-identical to the default mode, which is itself bit-exact against the
oracle (tests/test_gpu_parity.py); a sample is also checked against the oracle directly."""
import numpy as np
import pytest

from helpers import oracle_sums

pytestmark = pytest.mark.gpu

D = pytest.importorskip("paper_2405_14105_b200.dsi_sim")
from paper_2405_14105_b200 import workloads as W  # noqa: E402

SEED = W.SEED
MEANS = D.DSI_F_MEANS_ONLY
EXACT = ("trials", "nonsi_ticks", "sum_si_ticks", "sum_dsi_ticks", "sum_si_iters", "sum_accepts",
         "sum_segments", "threshold", "eq1_feasible", "min_lookahead", "mean_nonsi", "mean_si", "mean_dsi")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def results(cfgs, tick, flags=0, **kw):
    with D.Simulator(cfgs, tick=tick, seed=SEED, flags=flags, **kw) as sim:
        return sim.run().reduce(), sim.run().heatmap()


def assert_same_sums(got, want, ctx=""):
    for f in EXACT:
        assert np.array_equal(got[f], want[f]), (ctx, f)
    assert (got["sumsq_si_ticks"] == 0).all() and (got["sumsq_dsi_ticks"] == 0).all()
    assert np.isnan(got["std_si"]).all() and np.isnan(got["std_dsi"]).all()
    assert (got["n_dsi_gt_nonsi"] == -1).all() and (got["n_dsi_gt_si"] == -1).all()


def assert_cells_equal(a, b, ctx=""):
    for f in a.dtype.names:
        x, y = a[f], b[f]
        if x.dtype.kind == "f":
            assert np.array_equal(np.isnan(x), np.isnan(y)) and np.array_equal(x[~np.isnan(x)], y[~np.isnan(y)]), (ctx, f)
        else:
            assert np.array_equal(x, y), (ctx, f)


@pytest.mark.parametrize("name", ["fuzz", "cfg2", "cfg3", "cfg4", "long", "maxn", "fresh", "ttft", "ttft_mixed"])
def test_sums_and_heatmap_bit_identical_to_default(name):
    flags = 0
    if name == "fuzz":
        cfgs, tick = W.fuzz(160, seed=11, trials=300)
    elif name == "cfg2":
        cfgs, tick = W.cfg2(trials=3000)
    elif name == "cfg3":
        cfgs, tick = W.cfg3(trials=500, k_max=200, cells=slice(1, 10100, 41))
    elif name == "cfg4":
        cfgs, tick = W.cfg4(trials=777)
    elif name == "long":  # N up to 8192 (shared-memory histograms, 64 KB)
        cfgs = W.rows([(1.0, 0.05, 0.9, 3, 7, 1000, 0, 257), (1.0, 0.3, 0.5, 2, 3, 4097, 1, 65),
                       (1.0, 0.1, 0.97, 5, 2, 8192, 2, 40), (1.0, 1.0, 0.0, 1, 1, 8192, 0, 9),
                       (1.0, 0.2, 1.0, 4, 2, 8192, 0, 9)])
        tick = 0.01
    elif name == "maxn":  # N above 8192 up to the ABI's 32768: global-memory histograms
        cfgs = W.rows([(1.0, 0.1, 0.9, 4, 3, 32768, 0, 40), (1.0, 0.5, 0.6, 1, 1, 20000, 5, 33),
                       (1.0, 0.05, 0.3, 2, 7, 8193, 1, 70), (1.0, 0.2, 0.0, 1, 2, 32768, 0, 3)])
        tick = 0.01
    elif name == "ttft":  # the Table-2 protocol with prefill (first forwards cost TTFT, R23)
        cfgs, tick = W.cfg2_ttft(trials=3000)
    elif name == "ttft_mixed":  # TTFT and plain configs sharing indicator groups, N up to 2000
        rows = []
        for i, (N, a) in enumerate([(50, 0.9), (300, 0.6), (2000, 0.8), (1, 0.5), (7, 0.0), (40, 1.0)]):
            for k in (1, 3, 8):
                rows.append((2.0, 0.3, a, k, 1 + i % 4, N, 0, 900, 0.0, 0.0))
                rows.append((2.0, 0.3, a, k, 1 + i % 4, N, 0, 900, 9.5, 1.1))
        cfgs = np.array(rows, dtype=W.CONFIG_DTYPE)
        tick = 0.1
    else:
        cfgs, tick = W.cfg4(trials=500)
        flags = D.DSI_F_FRESH_VERIFIER
    want, want_cells = results(cfgs, tick, flags)
    got, got_cells = results(cfgs, tick, flags | MEANS)
    assert_same_sums(got, want, name)
    assert_cells_equal(got_cells, want_cells, name)


def test_sample_against_oracle():
    cfgs, tick = W.cfg3(trials=300, k_max=20, cells=slice(5, 10100, 401))
    got, _ = results(cfgs, tick, MEANS)
    for i in range(0, cfgs.size, 7):
        want = oracle_sums(cfgs[i], tick, SEED)
        assert int(got[i]["sum_dsi_ticks"]) == want["sum_dsi"] and int(got[i]["sum_si_ticks"]) == want["sum_si"]
        assert int(got[i]["sum_segments"]) == want["sum_m"] and int(got[i]["sum_accepts"]) == want["sum_acc"]


@pytest.mark.parametrize("kw", [{"n_shards": 3}, {"n_shards": 11}, {"nccl": True}, {"n_shards": 5, "ttft": True},
                                {"nccl": True, "ttft": True}])
def test_partition_and_one_rank_nccl(kw):
    kw = dict(kw)
    if kw.pop("ttft", False):  # the TTFT list split across the parts' config ranges
        cfgs, tick = W.cfg2_ttft(trials=2000)
    else:
        cfgs, tick = W.cfg3(trials=700, k_max=20, cells=slice(2, 10100, 97))
    want, want_cells = results(cfgs, tick, MEANS)
    extra = {"nccl_id": D.dsi_nccl_unique_id()} if kw.get("nccl") else kw
    got, got_cells = results(cfgs, tick, MEANS, **extra)
    for f in EXACT:
        assert np.array_equal(got[f], want[f]), f
    assert_cells_equal(got_cells, want_cells)


def test_update_keeps_groups_or_refuses():
    cfgs, tick = W.cfg3(trials=400, k_max=10, cells=slice(0, 10100, 211))
    other = cfgs.copy()
    other["lookahead"] = np.maximum(1, 11 - other["lookahead"])  # same indicator groups
    other["t_drafter"] = np.round(np.minimum(1.0, other["t_drafter"] * 2), 2)
    with D.Simulator(cfgs, tick=tick, seed=SEED, flags=MEANS) as sim:
        sim.run().reduce()
        got = sim.update(other).run().reduce()
        want, _ = results(other, tick, 0)
        for f in EXACT:
            assert np.array_equal(got[f], want[f]), f
        bad = other.copy()
        bad["accept_rate"][0] = 0.333  # a new indicator group
        with pytest.raises(D.DsiError) as e:
            sim.update(bad)
        assert e.value.status == D.DSI_E_RANGE
        again = sim.run().reduce()  # the handle keeps `other`
        for f in EXACT:
            assert np.array_equal(again[f], want[f]), f


def test_options_validated():
    cfgs, tick = W.fuzz(8, seed=3, trials=20)
    for flags in (D.DSI_F_PER_TRIAL, D.DSI_F_HIST, D.DSI_F_PATTERN, D.DSI_F_SHARED_STREAMS):
        with pytest.raises(D.DsiError) as e:
            D.Simulator(cfgs, tick=tick, seed=SEED, flags=MEANS | flags)
        assert e.value.status == D.DSI_E_RANGE


def test_exact_expectation_at_2_pow_32_trials():
    """n_trials = 2^32 per config (every value of the trial counter word) is cheap in this mode:
    the means sit within 6 sigma / sqrt(T) of the exact expectations (P11; tests/exact_math.py),
    sigma taken from a 2e6-trial default run -- a relative resolution of ~1e-5."""
    import math
    from fractions import Fraction

    import exact_math as X
    T = 1 << 32
    rows = [(1.0, 0.1, 0.8, 5, 2, 50, 0, T), (1.0, 0.3, 0.5, 3, 7, 100, 0, T)]
    got, _ = results(W.rows(rows), 0.01, MEANS)
    small = W.rows([r[:7] + (2_000_000,) for r in rows])
    ref, _ = results(small, 0.01, 0)
    for i, (tt, td, a, k, sp, N, _, _) in enumerate(rows):
        p = Fraction(int(got[i]["threshold"]), 2 ** 32)
        e = X.expectations(N, k, round(td * 100), round(tt * 100), sp, p)
        assert int(got[i]["trials"]) == T
        for mean, std, ex in ((got[i]["mean_dsi"], ref[i]["std_dsi"], e["dsi"]),
                              (got[i]["mean_si"], ref[i]["std_si"], e["si"])):
            assert abs(float(mean) / 0.01 - float(ex)) < 6 * (float(std) / 0.01) / math.sqrt(T), (i, mean, ex)


def test_full_heatmap_at_1e6_trials_against_exact_expectations():
    """The whole paper grid (10 100 cells x k 1..200 = 2.02e6 configs, N = 100) at 1e6 trials per
    config -- cheap in this mode -- against the exact expectations (tests/exact_math.py): every
    per-config SI and DSI mean within 7 sigma / sqrt(T) (sigma from a 1e4-trial default run), and
    Fig. 3(a)'s boundary on every cell whose exact SI/non-SI ratio is not within noise of 1."""
    from test_heatmap import exact_results
    cfgs, tick = W.cfg3()
    ref, _ = results(cfgs, tick, 0)           # 1e4 trials: per-config std
    big = cfgs.copy()
    big["n_trials"] = 1_000_000
    got, cells = results(big, tick, MEANS)
    ex = exact_results(cfgs, tick)
    T = 1_000_000
    for f, sf in (("mean_si", "std_si"), ("mean_dsi", "std_dsi")):
        tol = 7.0 * ref[sf] / np.sqrt(T) + 1e-9 * ex[f]
        err = np.abs(got[f] - ex[f])
        assert np.all(err <= tol), (f, int(np.argmax(err - tol)), float(np.max(err / np.maximum(tol, 1e-300))))
    exact_cells = D.dsi_heatmap(cfgs, ex)
    faster = cells["r_nonsi_si"] > 1.0
    expect = exact_cells["accept_rate"] > exact_cells["t_drafter"] / exact_cells["t_target"]
    # a cell may flip only if its exact non-SI/SI ratio is within 1e-3 of 1 (MC noise at 1e6 trials)
    near = np.abs(exact_cells["r_nonsi_si"] - 1.0) < 1e-3
    assert np.array_equal(faster[~near], expect[~near])
    assert np.all(cells["r_nonsi_dsi"] >= 1.0 - 1e-3)


def test_degenerate_sizes_every_mode():
    """n_trials = 1 and N in {1, 2, 33} with a in {0, 0.5, 1}: the default, shared-stream and
    means-only modes give the oracle's sums (one trial per config, one-token runs, a = 0 / 1 groups)."""
    from helpers import oracle_sums
    rows = []
    for N in (1, 2, 33):
        for a in (0.0, 0.5, 1.0):
            for k in (1, 4):
                rows.append((1.0, 0.2, a, k, 3, N, 0, 1))
    cfgs = W.rows(rows)
    outs = {}
    for name, flags in (("default", 0), ("shared", D.DSI_F_SHARED_STREAMS), ("means", MEANS)):
        outs[name], _ = results(cfgs, 0.01, flags)
    for i, row in enumerate(cfgs):
        want = oracle_sums(row, 0.01, SEED)
        for name, got in outs.items():
            assert int(got[i]["sum_dsi_ticks"]) == want["sum_dsi"], (name, i)
            assert int(got[i]["sum_si_ticks"]) == want["sum_si"], (name, i)
            assert int(got[i]["sum_segments"]) == want["sum_m"], (name, i)

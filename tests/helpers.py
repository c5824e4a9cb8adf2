"""Test helpers: turn a dsi_config row into the oracle's integer-tick Config."""
import numpy as np

import oracle as O


def oracle_config(row, tick: float, fresh: bool = False, halves: bool = False) -> O.Config:
    names = row.dtype.names
    tt1 = float(row["ttft_target"]) if "ttft_target" in names else 0.0
    td1 = float(row["ttft_drafter"]) if "ttft_drafter" in names else 0.0
    return O.Config(O.ticks(float(row["t_target"]), tick), O.ticks(float(row["t_drafter"]), tick),
                    float(row["accept_rate"]), int(row["lookahead"]), int(row["sp_degree"]),
                    int(row["n_tokens"]), int(row["stream_id"]),
                    O.ticks(tt1, tick) if tt1 else 0, O.ticks(td1, tick) if td1 else 0,
                    fresh_verifier=fresh, rng_halves=halves)


def oracle_sums(row, tick: float, seed: int, first: int = 0, count=None, pattern=False, hist=False,
                per_trial=False, fresh=False, halves=False):
    T = int(row["n_trials"]) if count is None else count
    return O.run(oracle_config(row, tick, fresh, halves), seed, first, T, pattern=pattern, hist=hist,
                 per_trial=per_trial)


RESULT_VS_ORACLE = (("sum_dsi_ticks", "sum_dsi"), ("sum_si_ticks", "sum_si"),
                    ("sumsq_dsi_ticks", "sumsq_dsi"), ("sumsq_si_ticks", "sumsq_si"),
                    ("sum_si_iters", "sum_iters"), ("sum_accepts", "sum_acc"),
                    ("sum_segments", "sum_m"), ("n_dsi_gt_nonsi", "n_dsi_gt_nonsi"),
                    ("n_dsi_gt_si", "n_dsi_gt_si"), ("trials", "trials"), ("nonsi_ticks", "nonsi"))


def assert_result_equals_oracle(res_row, want: dict, tick: float, ctx=""):
    for mine, theirs in RESULT_VS_ORACLE:
        assert int(res_row[mine]) == int(want[theirs]), (ctx, mine, int(res_row[mine]), want[theirs])
    m = O.means(want, tick)
    for k in ("mean_si", "mean_dsi", "mean_nonsi"):
        # north_star: FP64 means within 1e-9 relative (here both sides divide the same integers)
        assert abs(float(res_row[k]) - m[k]) <= 1e-9 * abs(m[k]), (ctx, k, float(res_row[k]), m[k])


def assert_trials_equal(got: dict, want: dict, ctx=""):
    for key in ("acc", "m", "iters", "si", "dsi"):
        g = np.asarray(got[key], np.int64)
        w = np.asarray(want[key], np.int64)
        if not np.array_equal(g, w):
            bad = np.nonzero(g != w)[0][:5]
            raise AssertionError(f"{ctx} {key} differs at trials {bad.tolist()}: {g[bad]} vs {w[bad]}")

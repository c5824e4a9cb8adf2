"""SPEC.md acceptance criterion 8 against the paper's printed Table 2:
DSI-vs-SI speedups of the ten (target, drafter, dataset) rows under the protocol of P:273
(50 tokens, prefill included, lookahead in {1, 5, 10}, DSI only on Eq.-1-feasible lookaheads at
SP 7), in exact expectation under this build's DSI reading.

The criterion's second half (every speedup > 1) holds.  Its first half (within +-20% of the
paper's 1.29-1.92x) does NOT: this reading gives 1.14-1.45x (DESIGN.md 3.1 explains why no
schedule that drafts every token can reach the paper's 1.92x for StarCoder/HumanEval).  The
miss is recorded as a strict xfail, so it stays visible and a change that fixes it is noticed."""
from fractions import Fraction

import pytest

import exact_math as X
from paper_2405_14105_b200 import workloads as W

# P:258-267, column "Speedup DSI vs. SI", in TABLE2_ROWS order
PAPER_SPEEDUP = [1.92, 1.66, 1.60, 1.41, 1.39, 1.37, 1.47, 1.41, 1.29, 1.70]


def protocol_speedups():
    """P:273 in exact expectation: ticks of 0.001 ms, TTFT = Table-3 ratio x TPOT."""
    cfgs, tick = W.cfg2_ttft(trials=1)
    out = []
    for i in range(len(W.TABLE2_ROWS)):
        rows = cfgs[3 * i:3 * i + 3]
        si, dsi = [], []
        for r in rows:
            t_t, t_d = round(r["t_target"] / tick), round(r["t_drafter"] / tick)
            t_t1, t_d1 = round(r["ttft_target"] / tick), round(r["ttft_drafter"] / tick)
            k, sp, n = int(r["lookahead"]), int(r["sp_degree"]), int(r["n_tokens"])
            a = Fraction(int(float(r["accept_rate"]) * 2 ** 32), 2 ** 32)
            e = X.expectations_ttft(n, k, t_d, t_t, sp, a, t_t1, t_d1)
            si.append(e["si"])
            if -(-t_t // (k * t_d)) <= sp:  # Eq. 1 at SP 7
                dsi.append(e["dsi"])
        out.append(float(min(si) / min(dsi)))
    return out


def test_criterion8_every_speedup_above_one():
    s = protocol_speedups()
    assert len(s) == 10 and min(s) > 1.0
    assert 1.10 < min(s) and max(s) < 1.50  # the 1.14-1.45x of DESIGN.md 3.1


@pytest.mark.xfail(strict=True, reason="SPEC criterion 8 (S:582) unmet: this DSI reading's offline speedups "
                                       "are 1.14-1.45x against the paper's 1.29-1.92x (DESIGN.md 3.1)")
def test_criterion8_within_20_percent_of_the_paper():
    s = protocol_speedups()
    assert all(abs(x - p) <= 0.2 * p for x, p in zip(s, PAPER_SPEEDUP)), list(zip(s, PAPER_SPEEDUP))

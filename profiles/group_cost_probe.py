"""Shared-stream kernel time of each acceptance-rate group of cfg3 alone (developer tool): the
check of the sharder's shared-stream cost model (dsi_validate.cpp shared_eval_cost, restated
below) on the heatmap's real groups -- 100 t_d x k 1..200 configs of one a each."""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402


def model(n, a, k):  # shared_eval_cost, two-pass form, per trial (ps)
    keff = min(k, n)
    stream = 0 < a < 1
    runs = 0 if (a == 0 or keff + 1 > n) else min(n / (keff + 1), (n * (1 - a) + 1) * a ** (keff + 1))
    p_any = 1 - math.exp(-runs)
    ln = min(n, 1 / (1 - a)) if a < 1 else n
    one = keff == 1
    return (n * (0.0040 + (0.00011 if stream else 0)) + p_any * ((1.78 if one else 2.43) + 0.0063 * ln)
            + runs * (0.143 if one else 0.68))


cfgs, tick = W.cfg3()
a100 = np.round(cfgs["accept_rate"] * 100).astype(int)
step = int(sys.argv[1]) if len(sys.argv) > 1 else 1
mult = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for ai in range(0, 101, step):
    sub = cfgs[a100 == ai].copy()
    sub["n_trials"] *= mult  # (longer launches: the per-launch fixed time and tail amortized)
    with D.Simulator(sub, tick=tick, seed=W.SEED, flags=D.DSI_F_TIMING | D.DSI_F_SHARED_STREAMS) as sim:
        sim.run()
        ms = []
        for _ in range(3):
            sim.run()
            ms.append(sim.kernel_ms())
    trials = sub["n_trials"].astype(np.int64)
    pred = sum(int(t) * (model(int(n), float(a), int(k)) + (1.3 if 0 < a < 1 else 0.05) * n / len(sub))
               for t, n, a, k in zip(trials, sub["n_tokens"], sub["accept_rate"], sub["lookahead"]))
    print(json.dumps({"a": ai / 100, "configs": len(sub), "ms": statistics.median(ms), "model_ms": pred * 1e-9}),
          flush=True)

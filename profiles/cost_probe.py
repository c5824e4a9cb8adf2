"""Kernel time per trial-token of single configs (developer tool): the data behind the sharder's
cost model (dsi_validate.cpp unit_cost, dsi_plan.cpp shared-stream unit costs).  Each probe is
a grid of identical-shape configs (same a, k, N) so the launch fills the GPU."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402

shared = "--shared" in sys.argv
rows_out = []
for N in (100, 1000):
    for a in (0.0, 0.01, 0.1, 0.3, 0.5, 0.7, 0.9, 0.99, 1.0):
        for k in (1, 2, 5, 20, 200):
            # launches of >= ~1 ms, so the per-launch fixed time and tail do not bias cheap points
            # (the first shared-stream probe, 2000 x 10^4, ran 0.03 ms kernels at a = 0)
            n_cfg = (20000 if N == 100 else 2000) if shared else (2000 if N == 100 else 200)
            trials = 40_000
            # t_d spread over 1..100 ticks (t_t = 100), SP 7: the heatmap's mix of queueing
            t_d = (np.arange(n_cfg) % 100 + 1) / 100.0
            rows = [(1.0, float(t_d[i]), a, k, 7, N, 0, trials) for i in range(n_cfg)]
            cfgs = W.rows(rows)
            flags = D.DSI_F_TIMING | (D.DSI_F_SHARED_STREAMS if shared else 0)
            with D.Simulator(cfgs, tick=0.01, seed=W.SEED, flags=flags) as sim:
                sim.run()
                ms = []
                for _ in range(3):
                    sim.run()
                    ms.append(sim.kernel_ms())
            tt = n_cfg * trials * N
            r = {"N": N, "a": a, "k": k, "ns_per_ktt": float(np.median(ms)) * 1e6 / (tt / 1e3)}
            rows_out.append(r)
            print(json.dumps(r), flush=True)

"""Projected strong scaling from measured shards (developer tool; not a bench number).

Every GPU box here has one B200, so the G-GPU run cannot be timed.  What the G ranks would each
do can: for G in 1, 2, 4, 8 this script creates the G rank handles of a workload one after the
other on the one GPU (world = G, rank = r; the test build's host transport stands in for NCCL and
is never called, since only dsi_sim_run is timed), runs each rank's share of the units and takes
its kernel time (CUDA events, DSI_F_TIMING).  The projected G-GPU kernel time is the slowest
rank's; the exchange step (one all-reduce of the per-config moments, or of the cells) is not
included.  Efficiency = T_1 / (G * max_r T_r): the quality of the cost-balanced (and cell-aligned)
partition on real kernels.

    python profiles/shard_projection.py [cfg3|cfg5] [--shared]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "cfg3"
flags = D.DSI_F_TIMING | (D.DSI_F_SHARED_STREAMS if "--shared" in sys.argv else 0)
cfgs, tick = W.cfg3() if name == "cfg3" else W.cfg5(D.dsi_min_lookahead)
tt = int(np.sum(cfgs["n_trials"].astype(np.int64) * cfgs["n_tokens"]))
D.select_library("test")
D.dsi_set_host_allreduce(lambda words: None)  # (never called: no reduce here)
out = {"workload": name, "shared_streams": bool(flags & D.DSI_F_SHARED_STREAMS), "trial_tokens": tt, "G": {}}
t1 = None
for G in (1, 2, 4, 8):
    per_rank = []
    for r in range(G):
        with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags, rank=r, world=G) as sim:
            sim.run()  # warm-up
            ms = []
            for _ in range(3):
                sim.run()
                ms.append(sim.kernel_ms())
            per_rank.append(statistics.median(ms))
            exchange = sim.comm_info()["heatmap_exchange"] if G > 1 else None
    tmax = max(per_rank)
    t1 = t1 or tmax
    out["G"][G] = {"rank_kernel_ms": per_rank, "max_ms": tmax, "projected_trial_tokens_per_s": tt / (tmax / 1e3),
                   "speedup": t1 / tmax, "efficiency": t1 / (G * tmax), "heatmap_exchange": exchange}
    print(json.dumps({"G": G, "max_ms": tmax, "speedup": t1 / tmax, "efficiency": t1 / (G * tmax)}), flush=True)
print(json.dumps(out))

"""A/B timing of trial-kernel builds and launch shapes on a cfg3 subsample.

    DSI_SIM_LIB=build/libX.so python profiles/ab.py --stride 5 --threads 128 --runs 5

Prints one JSON line: kernel ms per run (CUDA events around the trial kernel,
DSI_F_TIMING) and trial-tokens/s.  Developer tool; bench.py is the contract.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--stride", type=int, default=5)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--runs", type=int, default=5)
ap.add_argument("--shared", action="store_true", help="DSI_F_SHARED_STREAMS")
ap.add_argument("--fresh", action="store_true", help="DSI_F_FRESH_VERIFIER")
ap.add_argument("--halves", action="store_true", help="DSI_F_RNG_HALVES")
args = ap.parse_args()
if args.workload == "cfg3":
    cfgs, tick = W.cfg3(cells=slice(None, None, args.stride))
elif args.workload == "cfg5":
    cfgs, tick = W.cfg5(D.dsi_min_lookahead)
    cfgs = cfgs[:: args.stride]
elif args.workload == "cfg4":
    cfgs, tick = W.cfg4()
else:
    cfgs, tick = W.cfg2()
tt = int(np.sum(cfgs["n_trials"].astype(np.int64) * cfgs["n_tokens"]))
with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=D.DSI_F_TIMING | (D.DSI_F_SHARED_STREAMS if args.shared else 0)
                 | (D.DSI_F_FRESH_VERIFIER if args.fresh else 0) | (D.DSI_F_RNG_HALVES if args.halves else 0),
                 block_threads=args.threads) as sim:
    sim.run()
    sim.reduce()
    ms = []
    for _ in range(args.runs):
        sim.run()
        ms.append(sim.kernel_ms())
    res = sim.reduce()
print(json.dumps({"lib": os.environ.get("DSI_SIM_LIB", "default"), "workload": args.workload,
                  "shared": args.shared, "halves": args.halves,
                  "stride": args.stride, "threads": args.threads, "kernel_ms": ms,
                  "tt_per_s": tt / (statistics.median(ms) / 1e3),
                  "checksum": int(res["sum_dsi_ticks"].sum() % (1 << 61))}))

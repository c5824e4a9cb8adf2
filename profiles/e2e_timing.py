"""Where the e2e step's time goes (developer tool): update / run / reduce, host wall clock."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402

shared = "--shared" in sys.argv
means = "--means" in sys.argv
cfgs, tick = W.cfg3()
flags = (D.DSI_F_SHARED_STREAMS if shared else 0) | (D.DSI_F_MEANS_ONLY if means else 0)
out = {"shared": shared, "means": means}
with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
    res = np.zeros(cfgs.size, D.RESULT_DTYPE)
    sim.run().reduce(res)
    ts = {"update": [], "run": [], "reduce": []}
    for _ in range(4):
        t0 = time.perf_counter()
        sim.update(cfgs)
        t1 = time.perf_counter()
        sim.run()
        sim.heatmap()  # blocks: run + all-reduce + cells
        t2 = time.perf_counter()
        sim.reduce(res)  # all-reduce again + D2H + finalize
        t3 = time.perf_counter()
        ts["update"].append((t1 - t0) * 1e3)
        ts["run"].append((t2 - t1) * 1e3)
        ts["reduce"].append((t3 - t2) * 1e3)
    out.update({k + "_ms": statistics.median(v) for k, v in ts.items() if v})
print(json.dumps(out))

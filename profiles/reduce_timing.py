"""Where dsi_sim_reduce's time goes on the bench workload (developer tool).

Prints: the run alone, run + reduce, run + heatmap (no moment D2H), and a plain pinned
D2H of the moment table's size with torch, all host wall clock after a device sync.
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402

cfgs, tick = W.cfg3()
out = {}
with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=D.DSI_F_SHARED_STREAMS) as sim:
    res = np.zeros(cfgs.size, D.RESULT_DTYPE)
    cells = None
    for _ in range(3):
        sim.run().reduce(res)
        cells = sim.heatmap(cells)

    def t(fn, n=5):
        xs = []
        for _ in range(n):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            xs.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(xs)

    out["run_ms"] = t(lambda: sim.run())
    out["run_reduce_ms"] = t(lambda: sim.run().reduce(res))
    out["run_heatmap_ms"] = t(lambda: sim.run().heatmap(cells))
    sim.run()
    torch.cuda.synchronize()
    out["reduce_only_ms"] = t(lambda: sim.reduce(res))
dev = torch.empty(cfgs.size * 64, dtype=torch.uint8, device="cuda")
host = torch.empty(cfgs.size * 64, dtype=torch.uint8, pin_memory=True)
out["d2h_129MB_ms"] = t(lambda: host.copy_(dev, non_blocking=True))
out["host_threads"] = os.cpu_count()
print(json.dumps(out))

"""Shared-stream mode, one rank's share vs the whole (developer tool): creates the G = 1 handle
and the G = 2 / 8 rank handles of cfg3 (test build's host transport, never called), runs each
once -- for an ncu launch list of pass 1 / pass 2 per rank -- and prints each handle's unit
range and kernel time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402

cfgs, tick = W.cfg3()
D.select_library("test")
D.dsi_set_host_allreduce(lambda words: None)
flags = D.DSI_F_TIMING | D.DSI_F_SHARED_STREAMS
reps = int(os.environ.get("REPS", "3"))
for G, ranks in ((1, (0,)), (2, (0, 1)), (8, (0, 4))):
    for r in ranks:
        with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags, rank=r, world=G) as sim:
            ms = []
            for _ in range(reps):
                sim.run()
                ms.append(sim.kernel_ms())
            print(json.dumps({"G": G, "rank": r, "units": list(D.dsi_sim_units(sim.h)), "ms": ms,
                              "launches": sim.launches()}), flush=True)

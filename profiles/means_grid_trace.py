import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2405_14105_b200 import dsi_sim as D, workloads as W
cfgs, tick = W.cfg3()
with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=D.DSI_F_MEANS_ONLY | D.DSI_F_TIMING) as sim:
    out = None
    for i in range(6):
        t = time.perf_counter()
        sim.run()
        out = sim.heatmap(out)
        w = time.perf_counter() - t
        print(f"grid {w*1e3:.3f} ms kernel {sim.kernel_ms():.3f} ms", flush=True)

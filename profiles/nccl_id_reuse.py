import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2405_14105_b200 import dsi_sim as D, workloads as W
cfgs, tick = W.cfg1(trials=1000)
nid = D.dsi_nccl_unique_id()
with D.Simulator(cfgs, tick=tick, seed=1, nccl_id=nid) as a:
    a.run(); a.reduce()
print("first handle ok", flush=True)
t = time.time()
try:
    with D.Simulator(cfgs, tick=tick, seed=1, nccl_id=nid) as b:
        b.run(); b.reduce()
    print("second handle with the same id ok", time.time() - t, flush=True)
except D.DsiError as e:
    print("second handle failed:", e, time.time() - t, flush=True)

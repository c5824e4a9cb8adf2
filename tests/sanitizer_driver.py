"""Tiny runs of every kernel variant, for compute-sanitizer (tests/test_sanitizer.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402

cfgs, tick = W.fuzz(12, seed=9, trials=150)
for flags in (0, D.DSI_F_PER_TRIAL | D.DSI_F_HIST, D.DSI_F_SHARED_STREAMS):
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
        sim.run().reduce()
pat, _ = W.fuzz(4, seed=2, trials=64)
pat["n_tokens"] = 9
pat["n_trials"] = 256
pat["lookahead"] = 3
with D.Simulator(pat, tick=1.0, seed=W.SEED, flags=D.DSI_F_PATTERN | D.DSI_F_PER_TRIAL) as sim:
    sim.run().reduce()
long_n, _ = W.cfg1(trials=40)
long_n["n_tokens"] = 5000  # the arithmetic (non-table) variant
with D.Simulator(long_n, tick=0.01, seed=W.SEED) as sim:
    sim.run().reduce()
print("sanitizer driver ok")

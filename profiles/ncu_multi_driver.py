"""One dsi_multi_simulate launch of the multi-drafter heatmap, for an ncu capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_14105_b200 import dsi_sim as D, workloads as W  # noqa: E402

a_fast = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
cfgs, tick = W.multi_heatmap(a_fast=a_fast)
D.dsi_multi_simulate(cfgs, tick=tick, seed=W.SEED)

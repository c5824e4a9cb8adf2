"""Kernel time (CUDA events, DSI_F_TIMING) of dsi_multi_simulate on the multi-drafter heatmap
(W.multi_heatmap: cfg3's grid as drafter f_2 behind a fast drafter f_1), for two f_1
acceptance rates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time  # noqa: E402

import numpy as np  # noqa: E402

from paper_2405_14105_b200 import dsi_sim as D, workloads as W  # noqa: E402

HALVES = D.DSI_F_RNG_HALVES if "--halves" in sys.argv else 0
for a_fast in (0.5, 0.9):
    cfgs, tick = W.multi_heatmap(a_fast=a_fast)
    tt = int((cfgs["n_trials"].astype(np.int64) * cfgs["n_tokens"]).sum())
    for rep in range(4):
        t = time.perf_counter()
        D.dsi_multi_simulate(cfgs, tick=tick, seed=W.SEED, flags=D.DSI_F_TIMING | HALVES)
        w = time.perf_counter() - t
        ms, n = D.dsi_multi_last_kernel()
        print(f"multi_heatmap a_fast={a_fast}: kernel {ms:.3f} ms ({tt / ms * 1e3:.3e} trial-tokens/s), "
              f"wall {w * 1e3:.1f} ms, launches {n}")

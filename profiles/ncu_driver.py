"""One simulation of a (sub-sampled) bench workload, for ncu captures.

    ncu --set full --clock-control none --import-source on -k regex:dsi_trial_kernel -c 1 \
        -o gpurun_out/prof python profiles/ncu_driver.py --workload cfg3 --stride 10

--stride s keeps every s-th heatmap cell (all k of a kept cell), so the launch has the
same per-config mix as the full bench launch at 1/s of its length.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--stride", type=int, default=10)
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--shared", action="store_true", help="DSI_F_SHARED_STREAMS")
ap.add_argument("--means", action="store_true", help="DSI_F_MEANS_ONLY")
ap.add_argument("--halves", action="store_true", help="DSI_F_RNG_HALVES")
args = ap.parse_args()
if args.workload == "cfg3":
    cfgs, tick = W.cfg3(cells=slice(None, None, args.stride))
elif args.workload == "cfg5":
    cfgs, tick = W.cfg5(D.dsi_min_lookahead)
    cfgs = cfgs[:: args.stride]
else:
    raise SystemExit("workload")
flags = (D.DSI_F_SHARED_STREAMS if args.shared else 0) | (D.DSI_F_MEANS_ONLY if args.means else 0) | \
    (D.DSI_F_RNG_HALVES if args.halves else 0)
with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
    for _ in range(args.runs):
        sim.run()
        sim.reduce()
print(f"ran {cfgs.size} configs x {args.runs}")

"""Tiny runs of every kernel variant, for compute-sanitizer (tests/test_sanitizer.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2405_14105_b200 import dsi_sim as D  # noqa: E402
from paper_2405_14105_b200 import workloads as W  # noqa: E402

cfgs, tick = W.fuzz(12, seed=9, trials=150)
FRESH = D.DSI_F_FRESH_VERIFIER
for flags in (0, D.DSI_F_PER_TRIAL | D.DSI_F_HIST, D.DSI_F_SHARED_STREAMS, FRESH,
              FRESH | D.DSI_F_PER_TRIAL | D.DSI_F_HIST):
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
        sim.run().reduce()
        sim.heatmap()  # the on-device heatmap product
# the two-pass shared-stream form (groups of >= 256 configs): bulk copies on mbarriers
big, btick = W.cfg3(trials=300, k_max=8)
a100 = (big["accept_rate"] * 100).round().astype(int)
big = big[(a100 == 50) | (a100 == 90)].copy()
big["n_trials"] = 300 + 7 * (a100[(a100 == 50) | (a100 == 90)] == 90)
for flags in (D.DSI_F_SHARED_STREAMS, D.DSI_F_SHARED_STREAMS | FRESH):  # (FRESH: the template variant)
    with D.Simulator(big, tick=btick, seed=W.SEED, flags=flags) as sim:
        sim.run().reduce()
# cell-aligned shards: the heatmap kernel over an owned-cell index list; the deferred reduce
cells3, ctick3 = W.cfg3(trials=200, k_max=6, cells=slice(0, 60))
for flags in (0, D.DSI_F_SHARED_STREAMS):
    with D.Simulator(cells3, tick=ctick3, seed=W.SEED, flags=flags, n_shards=3) as sim:
        sim.run().heatmap()
        sim.run().reduce_device()
        sim.fetch(5, 20)
# the device path of dsi_sim_update (dsi_stage.cu): validate + convert on the GPU, commit, and a
# failing update (host path)
upd = cells3.copy()
upd["t_drafter"] = upd["t_drafter"] + 0.01
with D.Simulator(cells3, tick=ctick3, seed=W.SEED) as sim:
    sim.run().reduce()
    sim.update(upd).run().reduce()
    upd["t_drafter"][3] = 7.0
    try:
        sim.update(upd)
    except D.DsiError:
        pass
ttft, ttick = W.cfg2_ttft(trials=50)  # the TTFT variant (first-segment tables)
for flags in (0, D.DSI_F_PER_TRIAL | D.DSI_F_HIST, D.DSI_F_SHARED_STREAMS):
    with D.Simulator(ttft[:6], tick=ttick, seed=W.SEED, flags=flags) as sim:
        sim.run().reduce()
pat, _ = W.fuzz(4, seed=2, trials=64)
pat["n_tokens"] = 9
pat["n_trials"] = 256
pat["lookahead"] = 3
with D.Simulator(pat, tick=1.0, seed=W.SEED, flags=D.DSI_F_PATTERN | D.DSI_F_PER_TRIAL) as sim:
    sim.run().reduce()
# the arithmetic (non-table) variant; k t_d > t_t in the second row (fresh-verifier costs)
long_n = W.rows([(1.0, 0.1, 0.8, 5, 2, 5000, 0, 40), (1.0, 0.1, 0.8, 20, 2, 5000, 0, 40)])
for flags in (0, FRESH):
    with D.Simulator(long_n, tick=0.01, seed=W.SEED, flags=flags) as sim:
        sim.run().reduce()
# the k = 1 no-queue fast-path variant of the trial kernel (VAR 3), forced on
with D.use_library("checked" if os.environ.get("DSI_SIM_LIB") == "checked" else "test"):
    D.dsi_test_set_knob("k1_fast", 1)
    for flags in (0, D.DSI_F_PER_TRIAL):
        with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
            sim.run().reduce()
    D.dsi_test_set_knob("k1_fast", -1)
# means-only mode (dsi_seg.cu): histogram and evaluation passes, smem above 48 KB at N 8192
for flags in (D.DSI_F_MEANS_ONLY, D.DSI_F_MEANS_ONLY | FRESH):
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
        sim.run().reduce()
        sim.heatmap()
with D.Simulator(W.rows([(1.0, 0.1, 0.97, 5, 2, 8192, 2, 40), (1.0, 0.1, 0.5, 1, 2, 300, 0, 1000)]),
                 tick=0.01, seed=W.SEED, flags=D.DSI_F_MEANS_ONLY, n_shards=3) as sim:
    sim.run().reduce()
with D.Simulator(ttft[:9], tick=ttick, seed=W.SEED, flags=D.DSI_F_MEANS_ONLY, n_shards=2) as sim:
    sim.run().reduce()  # TTFT first-segment histograms and corrections
with D.Simulator(W.rows([(1.0, 0.1, 0.6, 3, 2, 9000, 0, 30)]), tick=0.01, seed=W.SEED,
                 flags=D.DSI_F_MEANS_ONLY) as sim:
    sim.run().reduce()  # global-memory histograms (N > 8192)
# multi-drafter kernel (dsi_multi.cu): D = 1, 2, 4, 7 variants, table and per-call q halves,
# pattern mode and per-trial records, ragged tiles
mf, mtick = W.multi_fuzz(20, seed=4, n_max=40, trials=70)
for flags in (0, D.DSI_F_PER_TRIAL, D.DSI_F_TIMING):
    D.dsi_multi_simulate(mf, tick=mtick, seed=W.SEED, flags=flags)
for m in (2, 3, 5, 8):
    rows = [(10.0, tuple(float(j + 1) for j in range(m - 1)), (0.5,) * (m - 1))]
    D.dsi_multi_simulate(W.multi_rows(rows, m ** 3, 4), tick=1.0, seed=W.SEED,
                         flags=D.DSI_F_PATTERN | D.DSI_F_PER_TRIAL)
D.dsi_multi_simulate(W.multi_rows([(1.0, (0.1, 0.3), (0.6, 0.8))], 2100, 5000), tick=0.01, seed=W.SEED)
# the halves layout (DSI_F_RNG_HALVES): every mode; thresholds whose high half is an f16 NaN pattern
# (XOR tie test) or 0 (all acceptances through ties), the pipelined walk (k >= 30), N > 4096
H = D.DSI_F_RNG_HALVES
hz = W.rows([(1.0, 0.1, a, k, 3, 100, 0, 300) for a in (0.49, 0.8, 2.0 ** -17) for k in (3, 40)])
hlong = W.rows([(1.0, 0.3, 0.5, 2, 3, 4097, 1, 65), (1.0, 0.1, 0.49, 40, 3, 4099, 0, 33)])
for grid in (hz, hlong, cfgs):
    for flags in (H, H | D.DSI_F_PER_TRIAL | D.DSI_F_HIST, H | FRESH):
        with D.Simulator(grid, tick=0.01 if grid is not cfgs else tick, seed=W.SEED, flags=flags) as sim:
            sim.run().reduce()
for grid, gt in ((hz, 0.01), (big, btick)):
    for flags in (H | D.DSI_F_SHARED_STREAMS, H | D.DSI_F_SHARED_STREAMS | FRESH, H | D.DSI_F_MEANS_ONLY):
        with D.Simulator(grid, tick=gt, seed=W.SEED, flags=flags) as sim:
            sim.run().reduce()
for flags in (H, H | D.DSI_F_PER_TRIAL, H | D.DSI_F_MEANS_ONLY):
    D.dsi_multi_simulate(mf, tick=mtick, seed=W.SEED, flags=flags)
D.dsi_multi_simulate(W.multi_rows([(1.0, (0.1, 0.3), (0.49, 0.8))], 700, 5000), tick=0.01, seed=W.SEED, flags=H)
print("sanitizer driver ok")

#!/usr/bin/env python
"""Benchmark of the DSI Monte Carlo latency simulator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3] [--impl ours|reference]

A step is one full pass of the hot path over the workload: dsi_sim_run (Philox ->
Bernoulli -> segment walk -> SI/DSI latencies -> per-config moments) followed by
dsi_sim_reduce (NCCL all-reduce across ranks, D2H, FP64 means).  The default
workload is BASELINE configs[2], the paper's heatmap: 100 drafter
latencies x 101 acceptance rates x k = 1..200 at SP 7, N = 100, 1e4 trials per
point = 2.02e6 configs, 2.02e12 trial-tokens.  Metric: simulated trial-tokens/s.

N > 1 runs one process per GPU under torch.distributed.run (the driver launches it
that way; `python bench.py --gpus N` without a torchrun environment re-executes itself
under torch.distributed.run with N processes); each rank simulates a cost-balanced
contiguous share of the (config, trial-tile) units and the per-config integer
moments are summed with one NCCL all-reduce inside dsi_sim_reduce.  Total work is
fixed as N grows, so the line reports "scaling": "strong".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2405_14105_b200 import workloads as W  # noqa: E402

METRIC = "simulated trial-tokens/sec"
UNIT = "trial-tokens/s"
SM_COUNT = 148
LANES_PER_SM_CLK = 4 * 32  # 4 SMSPs x 32 lanes issue one thread-instruction each per clock


def workload(name: str, min_lookahead):
    if name == "cfg1":
        return W.cfg1()
    if name == "cfg2":
        return W.cfg2()
    if name == "cfg3":
        return W.cfg3()
    if name == "cfg3-fast":
        return W.cfg3(k_max=20)
    if name == "cfg4":
        return W.cfg4()
    if name == "cfg5":
        return W.cfg5(min_lookahead)
    raise SystemExit(f"unknown workload {name}")


WORKLOAD_DESC = {
    "cfg1": "BASELINE configs[0]: single point t_t=1.0 t_d=0.1 a=0.8 k=5 SP=2 N=50, 1e3 trials",
    "cfg2": "BASELINE configs[1]: Table-2 pairs (P:258-267) x k{1,5,10}, SP=8, N=100, 1e5 trials",
    "cfg3": "BASELINE configs[2]: heatmap t_d 0.01..1.00 x a 0.00..1.00 x k 1..200, SP=7, N=100, 1e4 trials",
    "cfg3-fast": "heatmap with k 1..20 (BASELINE configs[2] fast variant)",
    "cfg4": "BASELINE configs[3]: k 1..20 x SP 2..8 at t_d=0.1 a=0.8, N=500, 1e5 trials",
    "cfg5": "BASELINE configs[4]: 10100 heatmap cells, k=Eq.1 min_lookahead, SP=7, N=1000, 1e5 trials",
}


def heatmap_grid_times(sim, flush, steps):
    """Wall time of run + on-device heatmap product per step (L2 flushed before each)."""
    import torch
    out, times = None, []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim.run()
        out = sim.heatmap(out)
        times.append(time.perf_counter() - t0)
    return times, out


def cells_equal(a, b) -> bool:
    if a.size != b.size:
        return False
    for f in b.dtype.names:
        x, y = a[f], b[f]
        if x.dtype.kind == "f":
            if not np.array_equal(x, y, equal_nan=True):
                return False
        elif not np.array_equal(x, y):
            return False
    return True


def fig_summary(cfgs, res, cells) -> dict:
    """The paper's heatmap claims on one run's results (rank 0): Fig. 3 (SI over all k,
    DSI over the Eq.-1-feasible k at SP 7) from the cells, and Fig. 5 (App. F.7; SI and
    DSI both at lookahead 5) from the k = 5 configs: the cells where SI is slower than non-SI
    (Fig. 5(a)'s pink) and where DSI is slower than SI or than non-SI ("DSI is never slower than
    either SI or non-SI")."""
    out = {"fig3": {"cells": int(cells.size),
                    "max_min_si_nonsi_over_dsi": float(np.nanmax(cells["r_min_dsi"])),
                    "cells_dsi_slower_than_si": int(np.sum(cells["r_si_dsi"] < 1.0)),
                    "cells_dsi_slower_than_nonsi": int(np.sum(cells["r_nonsi_dsi"] < 1.0))}}
    k5 = cfgs["lookahead"] == 5
    if np.any(k5):
        r = res[k5]
        out["fig5_k5"] = {"cells": int(np.sum(k5)),
                          "si_slower_than_nonsi": int(np.sum(r["mean_si"] > r["mean_nonsi"])),
                          "dsi_slower_than_si": int(np.sum(r["mean_dsi"] > r["mean_si"])),
                          "dsi_slower_than_nonsi": int(np.sum(r["mean_dsi"] > r["mean_nonsi"]))}
    return out


def fresh_verifier_block(D, cfgs, tick, base_kw, root, fresh_id, flush, steps, res_default) -> dict:
    """The fresh-verifier reading (R24, Thm 2's proof P:445) on the same workload: the
    per-config kernel once (its sums are the reference for the fast modes), then the
    shared-stream and means-only heatmap grid times; the fast modes' sums and cells must be
    bit-identical to the per-config R24 run, and every config with k t_d <= t_t identical to
    the default reading's."""
    flags = D.DSI_F_TIMING | D.DSI_F_FRESH_VERIFIER | root
    simf = D.Simulator(cfgs, flags=flags, nccl_id=fresh_id(), **base_kw)
    simf.run()
    resf = simf.reduce()
    kern_ms = simf.kernel_ms()
    simf.close()
    simfs = D.Simulator(cfgs, flags=flags | D.DSI_F_SHARED_STREAMS, nccl_id=fresh_id(), **base_kw)
    simfs.run()
    ress = simfs.reduce()
    heat_s, cells_s = heatmap_grid_times(simfs, flush, steps)
    simfs.close()
    simfm = D.Simulator(cfgs, flags=flags | D.DSI_F_MEANS_ONLY, nccl_id=fresh_id(), **base_kw)
    simfm.run()
    resm = simfm.reduce()
    heat_m, cells_m = heatmap_grid_times(simfm, flush, steps)
    simfm.close()
    out = {"reading": "R24 fresh verifier (DSI_F_FRESH_VERIFIER)",
           "per_config_kernel_ms": kern_ms,
           "grid_time_shared_streams_s": statistics.median(heat_s),
           "grid_time_means_only_s": statistics.median(heat_m)}
    if res_default is not None and resf.size:  # rank 0 (REDUCE_TO_ROOT)
        cells_f = D.dsi_heatmap(cfgs, resf)
        sums = ("sum_si_ticks", "sum_dsi_ticks", "sum_segments", "sum_si_iters", "trials")
        out["shared_streams_bit_identical"] = bool(
            all(np.array_equal(ress[f], resf[f]) for f in sums + ("sumsq_dsi_ticks", "n_dsi_gt_nonsi", "n_dsi_gt_si"))
            and cells_equal(cells_s, cells_f))
        out["means_only_bit_identical"] = bool(all(np.array_equal(resm[f], resf[f]) for f in sums)
                                               and cells_equal(cells_m, cells_f))
        # the readings differ only where k t_d > t_t (integer ticks)
        same = cfgs["lookahead"] * np.rint(cfgs["t_drafter"] / tick) <= np.rint(cfgs["t_target"] / tick)
        out["configs_where_readings_differ"] = int(np.sum(~same))
        out["identical_to_default_where_k_td_le_tt"] = bool(
            np.array_equal(resf["sum_dsi_ticks"][same], res_default["sum_dsi_ticks"][same]))
        out["trials_dsi_slower_than_nonsi"] = int(np.sum(resf["n_dsi_gt_nonsi"]))
        out["figures"] = fig_summary(cfgs, resf, cells_f)
    return out


def fast_mode_e2e(sim, cfgs, res, tt, steps, barrier, max_over_ranks):
    """End to end through the public API with host buffers, host wall clock, max over ranks:
    e2e = dsi_sim_update (H2D of the configs from pinned host memory, validated on the device) + run
    + dsi_sim_heatmap (the heatmap job's result: all-reduce, device argmin, D2H of the cells);
    e2e_all_results = update + run + dsi_sim_reduce of every config's result to the host."""
    h2d, d2h_all = sim.io_bytes()
    cells = None
    out = []
    sim.update(cfgs)  # (warm-up: buffers of the update path)
    for job in ("heatmap", "all"):
        barrier()
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            sim.update(cfgs)
            sim.run()
            if job == "heatmap":
                cells = sim.heatmap(cells)
            else:
                sim.reduce(res)
            ts.append(time.perf_counter() - t0)
        d2h = int(cells.nbytes) if job == "heatmap" else int(d2h_all)
        out.append({"value": tt * steps / max_over_ranks(sum(ts)), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": d2h,
                    "step": "update + run + heatmap (cells to the host)" if job == "heatmap"
                    else "update + run + reduce (every result to the host)"})
    return out[0], out[1]


def other_workloads_block(D, names, args, base_kw, root, fresh_id, flush, barrier, max_over_ranks, world) -> dict:
    """BASELINE.json's other configs on the same GPUs (collective: every rank runs its share):
    per workload the per-config mode (run + reduce, CUDA events, as `value`) with its SURVEY 8(d).4
    issue fraction, and the shared-stream and means-only modes (run + reduce_device) with whether
    their sums equal the per-config run's; and the per-config mode under the halves layout (R26)."""
    import torch

    sm_max = float(measured_peaks().get("sm_max_mhz", 1965.0))
    peak_instr = SM_COUNT * LANES_PER_SM_CLK * sm_max * 1e6
    out = {}
    for name in names:
        cfgs, tick = workload(name, D.dsi_min_lookahead)
        kw = dict(base_kw, tick=tick)
        tt = trial_tokens(cfgs)
        entry = {"desc": WORKLOAD_DESC[name], "configs": int(cfgs.size), "trial_tokens_per_step": tt}
        ref = None
        for mode, flags in (("per_config", 0), ("shared_streams", D.DSI_F_SHARED_STREAMS),
                            ("means_only", D.DSI_F_MEANS_ONLY), ("per_config_rng_halves", D.DSI_F_RNG_HALVES)):
            sim = D.Simulator(cfgs, flags=D.DSI_F_TIMING | root | flags, nccl_id=fresh_id(), **kw)
            st = torch.cuda.ExternalStream(sim.stream(), device=torch.device("cuda", base_kw["device"]))
            res = np.zeros(cfgs.size, D.RESULT_DTYPE)
            for _ in range(args.warmup):
                sim.run()
                sim.reduce(res)
            barrier()
            ms, kms = [], []
            for _ in range(args.steps):
                flush.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                sim.run()
                if flags & (D.DSI_F_SHARED_STREAMS | D.DSI_F_MEANS_ONLY):
                    sim.reduce_device()
                else:
                    sim.reduce(res)
                e1.record(st)
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
                kms.append(sim.kernel_ms())
            barrier()
            total = max_over_ranks(sum(ms))
            kern = max_over_ranks(statistics.mean(kms))
            d = {"value": tt * args.steps / (total / 1000.0), "unit": UNIT, "ms_per_step": total / args.steps,
                 "kernel_ms": kern}
            if flags == 0:
                ach = alg_instructions(cfgs) / world / (kern / 1000.0)
                d["roofline_issue_frac"] = ach / peak_instr
                ref = res
            elif flags == D.DSI_F_RNG_HALVES:  # the halves layout (R26): its own accounting, its own draws
                ach = alg_instructions_halves(cfgs) / world / (kern / 1000.0)
                d["roofline_issue_frac"] = ach / peak_instr
            elif base_kw["rank"] == 0:
                sim.fetch(0, cfgs.size, res)
                d["sums_identical_to_per_config"] = bool(all(
                    np.array_equal(res[f], ref[f]) for f in ("sum_si_ticks", "sum_dsi_ticks", "sum_segments",
                                                             "sum_si_iters", "trials")))
            sim.close()
            entry[mode] = d
        out[name] = entry
    return out


def alg_instructions_halves(cfgs) -> float:
    """As alg_instructions for the halves layout (DSI_F_RNG_HALVES, R26): Philox4x32-10
    serves 8 positions per call (40 instructions / 8 = 5 per trial-token), 1 compare, 10 per
    rejection; the tie-break call (probability 2^-16 per position) adds < 0.001 per token."""
    tt = cfgs["n_trials"].astype(np.float64) * cfgs["n_tokens"].astype(np.float64)
    return float(np.sum(tt * (6.0 + 10.0 * (1.0 - cfgs["accept_rate"]))))


def rng_halves_block(D, cfgs, cfgs_pinned, tick, args, base_kw, root, fresh_id, flush, barrier, max_over_ranks,
                     world, peak_instr) -> dict:
    """The same workload under the halves layout of the indicator stream (DSI_F_RNG_HALVES):
    the per-config mode timed exactly as `value` (run + reduce, CUDA events, L2 flushed), and
    the shared-stream and means-only modes (run + reduce_device) checked bit-identical to it."""
    import torch

    tt = trial_tokens(cfgs)
    out = {"layout": "DSI_F_RNG_HALVES (DESIGN.md R26): 16 bits per Bernoulli from Philox at (q, 0, trial, "
                     "stream), q = (p-1) >> 3, plus an exact tie-break draw at (q, 1, trial, stream) when the 16 "
                     "bits equal the threshold's high half: A_p = [v 2^16 + w < floor(a 2^32)], the same law as "
                     "`value`'s layout with half the Philox calls (different draws, so different sums)"}
    ref = None
    for mode, flags in (("per_config", 0), ("shared_streams", D.DSI_F_SHARED_STREAMS),
                        ("means_only", D.DSI_F_MEANS_ONLY)):
        sim = D.Simulator(cfgs, flags=D.DSI_F_TIMING | D.DSI_F_RNG_HALVES | root | flags, nccl_id=fresh_id(),
                          **dict(base_kw, tick=tick))
        st = torch.cuda.ExternalStream(sim.stream(), device=torch.device("cuda", base_kw["device"]))
        res = np.zeros(cfgs.size, D.RESULT_DTYPE)
        for _ in range(args.warmup):
            sim.run()
            sim.reduce(res)
        barrier()
        torch.cuda.synchronize()
        ms, kms = [], []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            sim.run()
            if flags:
                sim.reduce_device()
            else:
                sim.reduce(res)
            e1.record(st)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
            kms.append(sim.kernel_ms())
        barrier()
        total = max_over_ranks(sum(ms))
        kern = max_over_ranks(statistics.mean(kms))
        d = {"value": tt * args.steps / (total / 1000.0), "unit": UNIT, "ms_per_step": total / args.steps,
             "kernel_ms": kern, "launches_per_step": sim.launches()}
        if flags == 0:
            # end to end as `e2e`: update (configs from pinned host memory) + run + reduce to the host
            h2d, d2h = sim.io_bytes()
            sim.update(cfgs_pinned)
            sim.run()
            sim.reduce(res)
            barrier()
            ts = []
            for _ in range(args.steps):
                t0 = time.perf_counter()
                sim.update(cfgs_pinned)
                sim.run()
                sim.reduce(res)
                ts.append(time.perf_counter() - t0)
            d["e2e"] = {"value": tt * args.steps / max_over_ranks(sum(ts)), "unit": UNIT,
                        "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}
            ach = alg_instructions_halves(cfgs) / world / (kern / 1000.0)
            ncu_h = None  # --set full of one full bench launch of this kernel (profiles/, if captured)
            try:
                with open(os.path.join(ROOT, "profiles", "latest_halves_ncu_summary.json")) as f:
                    k = json.load(f)["kernels"][0]
                ncu_h = {"issue_active_pct": float(k["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
                         "fmaheavy_pct": float(
                             k["sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"][0]),
                         "alu_pct": float(k["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"][0]),
                         "registers": int(k["launch__registers_per_thread"][0]),
                         "source": "profiles/latest_halves_ncu_summary.json (" + json.load(open(
                             os.path.join(ROOT, "profiles", "latest_halves_ncu_summary.json")))["report"] + ")"}
            except (OSError, KeyError, ValueError, IndexError):
                pass
            d["roofline"] = {"bound": "alu", "achieved": ach / 1e9, "peak": peak_instr / 1e9, "unit": "Ginstr/s",
                             "frac": ach / peak_instr, "kernel": "dsi_trial_kernel<..., HALVES>", "ncu": ncu_h,
                             "work": "6 + 10(1-a) thread-instructions per trial-token: 5 for Philox4x32-10 (40 "
                                     "per call of 8 indicators), 1 compare, 10 per rejection"}
            ref = res
        elif base_kw["rank"] == 0:
            sim.fetch(0, cfgs.size, res)
            fields = ("sum_si_ticks", "sum_dsi_ticks", "sum_segments", "sum_si_iters", "trials")
            if flags == D.DSI_F_SHARED_STREAMS:
                fields += ("sumsq_si_ticks", "sumsq_dsi_ticks", "n_dsi_gt_nonsi", "n_dsi_gt_si")
            d["sums_identical_to_per_config"] = bool(all(np.array_equal(res[f], ref[f]) for f in fields))
        # the heatmap product under this layout (run + dsi_sim_heatmap, host wall clock, as heatmap.grid_time_*)
        d["heatmap_grid_time_s"] = max_over_ranks(statistics.median(heatmap_grid_times(sim, flush, args.steps)[0]))
        sim.close()
        out[mode] = d
    if base_kw["rank"] == 0:
        a = cfgs["accept_rate"]
        acc = ref["sum_accepts"].astype(np.float64) / (cfgs["n_trials"] * (cfgs["n_tokens"] - 1.0))
        sd = np.sqrt(a * (1 - a) / (cfgs["n_trials"] * (cfgs["n_tokens"] - 1.0))) + 1e-12
        z = np.abs(acc - a) / sd
        _, first = np.unique(np.stack([cfgs["accept_rate"], cfgs["stream_id"].astype(np.float64),
                                       cfgs["n_tokens"].astype(np.float64), cfgs["n_trials"].astype(np.float64)]),
                             axis=1, return_index=True)
        zi = z[first]  # one per distinct indicator stream (configs of a group draw identical indicators)
        out["acceptance_law"] = {"streams": int(first.size), "max_abs_z": float(np.max(zi)),
                                 "mean_z2": float(np.mean(zi * zi)),
                                 "note": "per distinct (a, stream, N, T) -- every config of such a group draws the "
                                         "same indicators -- the realised acceptance fraction vs a in units of its "
                                         "binomial sd (mean z^2 ~ 1 for the exact law)"}
    return out


def trial_tokens(cfgs) -> int:
    return int(np.sum(cfgs["n_trials"].astype(np.int64) * cfgs["n_tokens"].astype(np.int64)))


def alg_instructions(cfgs) -> float:
    """Algorithmic thread-instructions of one pass: per trial-token
    10 (Philox4x32-10: 10 rounds x (2 mul-wide + 2 xor) / 4 words) + 1 (Bernoulli compare)
    + 10 per rejection (segment walk + SI/DSI cost), (1 - a) rejections per token."""
    tt = cfgs["n_trials"].astype(np.float64) * cfgs["n_tokens"].astype(np.float64)
    return float(np.sum(tt * (11.0 + 10.0 * (1.0 - cfgs["accept_rate"]))))


def alg_multiplies(cfgs) -> float:
    """Algorithmic 32x32->64 multiplies of one pass: Philox4x32-10 takes 10 rounds x 2 per
    call of 4 indicators, ceil((N-1)/4) calls per trial; configs with a = 0
    or a = 1 need no random numbers (thresholds 0 and 2^32)."""
    thr = np.floor(cfgs["accept_rate"] * 4294967296.0)
    rnd = (thr > 0) & (thr < 4294967296.0)
    calls = cfgs["n_trials"].astype(np.float64) * np.ceil((cfgs["n_tokens"].astype(np.float64) - 1) / 4)
    return float(np.sum(calls[rnd]) * 20.0)


def multi_alg_multiplies(cfgs) -> float:
    """Expected algorithmic multiplies of one multi-drafter pass (dsi_multi_simulate): the RNG
    contract gives drafter j's indicators of a quad from one Philox call (20 multiplies), and
    the call is needed only if the quad still has a position no earlier drafter settled:
    P = 1 - (1 - prod_{i<j}(1 - a_i))^r for a quad of r positions; a_j in {0, 1} needs none."""
    total = 0.0
    for c in cfgs:
        npos = int(c["n_tokens"]) - 1
        full, rem = divmod(npos, 4)
        open_p = 1.0
        calls = 0.0
        for j in range(int(c["n_drafters"])):
            thr = np.floor(c["accept_rate"][j] * 4294967296.0)
            a = thr / 4294967296.0
            if 0 < thr < 4294967296.0:
                calls += full * (1.0 - (1.0 - open_p) ** 4)
                if rem:
                    calls += 1.0 - (1.0 - open_p) ** rem
            open_p *= 1.0 - a
        total += float(c["n_trials"]) * calls * 20.0
    return total


def multi_drafter_block(steps: int, sm_max: float) -> dict:
    """Multi-drafter DSI on W.multi_heatmap: kernel time by CUDA events
    (DSI_F_TIMING) and the one-call host wall clock (config H2D + kernel + moments D2H)."""
    from paper_2405_14105_b200 import dsi_sim as D
    cfgs, tick = W.multi_heatmap()
    tt = int(np.sum(cfgs["n_trials"].astype(np.int64) * cfgs["n_tokens"]))
    D.dsi_multi_simulate(cfgs, tick=tick, seed=W.SEED, flags=D.DSI_F_TIMING)  # warm-up
    ks, ws = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        D.dsi_multi_simulate(cfgs, tick=tick, seed=W.SEED, flags=D.DSI_F_TIMING)
        ws.append(time.perf_counter() - t0)
        ks.append(D.dsi_multi_last_kernel()[0])
    k_ms = statistics.median(ks)
    # means-only: configs differing only in latencies share one pass (101 acceptance groups here)
    ms_means = []
    for _ in range(steps):
        D.dsi_multi_simulate(cfgs, tick=tick, seed=W.SEED, flags=D.DSI_F_TIMING | D.DSI_F_MEANS_ONLY)
        ms_means.append(D.dsi_multi_last_kernel()[0])
    mults = multi_alg_multiplies(cfgs)
    # the halves layout (R26): drafter j on counter word 1 = 2(j-1), 8 positions per call
    ms_h = []
    for _ in range(steps):
        D.dsi_multi_simulate(cfgs, tick=tick, seed=W.SEED, flags=D.DSI_F_TIMING | D.DSI_F_RNG_HALVES)
        ms_h.append(D.dsi_multi_last_kernel()[0])
    return {"workload": "W.multi_heatmap: m = 3, f_1 (t 0.01, a 0.5) ahead of cfg3's 10100 (t_d, a) "
                        "points as f_2, t_m 1.0, N 100, 1e4 trials, lookahead 1 (Alg. 1 as stated)",
            "value": tt / (k_ms / 1000.0), "unit": UNIT, "kernel_ms": k_ms,
            "trial_tokens_per_step": tt, "gpu_launches": D.dsi_multi_last_kernel()[1],
            "rng_halves": {"value": tt / (statistics.median(ms_h) / 1000.0), "unit": UNIT,
                           "kernel_ms": statistics.median(ms_h),
                           "note": "DSI_F_RNG_HALVES (DESIGN.md R26): 16 bits per indicator plus an exact "
                                   "tie-break draw, one Philox call per 8 positions and drafter"},
            "means_only": {"value": tt / (statistics.median(ms_means) / 1000.0), "unit": UNIT,
                           "kernel_ms": statistics.median(ms_means),
                           "note": "DSI_F_MEANS_ONLY: one pass per acceptance group, sums for every "
                                   "latency by linearity; same sums and means, no std"},
            "e2e": {"value": tt / statistics.median(ws), "unit": UNIT,
                    "h2d_bytes_per_step": int(cfgs.size * 112 + (cfgs.size + 1) * 8),
                    "d2h_bytes_per_step": int(cfgs.size * 11 * 8)},
            "roofline": {"bound": "alu", "achieved": mults / (k_ms / 1000.0) / 1e9,
                         "peak": mul_peak(sm_max) / 1e9, "unit": "Gmul/s",
                         "frac": mults / (k_ms / 1000.0) / mul_peak(sm_max), "kernel": "dsi_multi_kernel",
                         "work": "20 multiplies per Philox call a drafter must make (quads with an "
                                 "unsettled position), expected over the configs"}}


def imad_wide_cycles() -> float:
    """Cycles per warp-wide IMAD.WIDE.U32 on one SMSP, measured by profiles/pipe_peaks.cu (the
    Philox half round IMAD.WIDE + LOP3, profiles/r02_pipe_peaks.jsonl); 4.0 if the file is absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_pipe_peaks.jsonl")) as f:
            for ln in f:
                d = json.loads(ln)
                if d.get("op", "").startswith("IMAD.WIDE + LOP3"):
                    return 2.0 * float(d["cycles_per_warp_instr"])  # two instructions per step
    except (OSError, ValueError):
        pass
    return 4.0


def mul_peak(sm_mhz: float) -> float:
    """The fmaheavy pipe's 32x32->64 multiply rate: 148 SMs x 4 SMSPs x 32 lanes per IMAD.WIDE
    issue interval (measured, imad_wide_cycles)."""
    return SM_COUNT * 4 * 32 / imad_wide_cycles() * sm_mhz * 1e6


def _imad_ceiling(sm_mhz: float) -> float:
    """Trial-tokens/s if the fmaheavy pipe did nothing but Philox multiplies: the measured
    IMAD.WIDE rate, 16 per Philox call of 4 tokens (rounds 2-9; rounds 0-1 are hoisted)."""
    return mul_peak(sm_mhz) / 16.0 * 4.0


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle baseline
def _oracle_sample_configs(cfgs, tick, n=100):
    import oracle as O

    sub = W.subsample(cfgs, n)
    ocfgs = [O.Config(O.ticks(float(r["t_target"]), tick), O.ticks(float(r["t_drafter"]), tick),
                      float(r["accept_rate"]), int(r["lookahead"]), int(r["sp_degree"]),
                      int(r["n_tokens"]), int(r["stream_id"])) for r in sub]
    return sub, ocfgs


def _oracle_worker(job):
    """One host process of the multi-process oracle timing: trials [first, first + S) of every
    sampled config, started at a common wall-clock instant."""
    import oracle as O

    ocfgs, S, first, start_at = job
    O.run(ocfgs[0], W.SEED, first, 1, per_trial=False)  # load the library before the start
    while time.time() < start_at:
        time.sleep(0.001)
    t0 = time.time()
    tt = 0
    for c in ocfgs:
        O.run(c, W.SEED, first, S, per_trial=False)
        tt += S * c.n_tokens
    return tt, t0, time.time()


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_oracle_sample(cfgs, tick, seconds: float, processes: int = 1):
    """The oracle as it stands (single-threaded C) on a bounded sample of the workload: the
    first S trials of 100 evenly spaced configs per process, S sized to ~`seconds` of work.
    processes > 1: that many independent host processes on disjoint interleaved subsets of
    100 x processes evenly spaced configs, started together; value = all their trial-tokens
    / the common wall time."""
    import oracle as O

    sub, ocfgs = _oracle_sample_configs(cfgs, tick, 100 * processes)
    probe = ocfgs[::processes]
    t0 = time.perf_counter()  # calibrate: 2 trials of each config of one process's share
    for c in probe:
        O.run(c, W.SEED, 0, 2, per_trial=False)
    per_trial = (time.perf_counter() - t0) / (2 * len(probe))
    S = int(max(1, min(int(sub["n_trials"].min()), seconds / (per_trial * len(probe)))))
    if processes <= 1:
        tt, a, b = _oracle_worker((ocfgs, S, 0, 0.0))
        dt = b - a
    else:
        import multiprocessing as mp

        start_at = time.time() + 2.0 + 0.05 * processes
        with mp.get_context("spawn").Pool(processes) as pool:
            res = pool.map(_oracle_worker, [(ocfgs[w::processes], S, 0, start_at) for w in range(processes)])
        tt = sum(r[0] for r in res)
        dt = max(r[2] for r in res) - min(r[1] for r in res)
    return {"value": tt / dt, "unit": UNIT, "cores": processes, "kind": "oracle",
            "sample": f"first {S} trials of {len(ocfgs)} evenly spaced configs of the workload, "
                      f"{processes} process(es) on disjoint config subsets ({tt} trial-tokens, {dt:.1f} s "
                      f"wall; single-threaded C oracle: literal SI loop + DSI event simulation)"}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    O.build()
    cfgs, tick = workload(args.workload, _min_lookahead_plain)
    per_step = max(1.0, args.reference_seconds / max(1, args.steps + args.warmup))
    procs = host_cores()
    for _ in range(args.warmup):
        run_oracle_sample(cfgs, tick, per_step / 4, procs)
    vals = []
    t0 = time.perf_counter()
    last = None
    for _ in range(args.steps):
        last = run_oracle_sample(cfgs, tick, per_step, procs)
        vals.append(last["value"])
    wall = time.perf_counter() - t0
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * wall / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32/int64",
            "data": "synthetic", "config": {"workload": args.workload, "desc": WORKLOAD_DESC[args.workload]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "oracle",
                             "sample": last["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def _min_lookahead_plain(t_t, t_d, sp):
    k = 1
    while -(-t_t // (k * t_d)) > sp:
        k += 1
    return k


# ----------------------------------------------------------------------------- our arm
def ours(args):
    import torch
    import torch.distributed as dist

    from paper_2405_14105_b200 import dsi_sim as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:  # the library's NCCL communicator prints its rank count at init (stderr)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    # DSI_BENCH_ONE_GPU=1 (test mode, numbers meaningless): every rank on GPU 0, gloo process
    # group, the library's cross-rank sums through the host all-reduce hook -- exercises the
    # whole multi-rank flow on a one-GPU box (NCCL refuses two ranks on one GPU)
    one_gpu = world > 1 and os.environ.get("DSI_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    elif local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local} but {torch.cuda.device_count()} are visible")
    torch.cuda.set_device(local)
    coll_dev = "cpu" if one_gpu else "cuda"
    if world > 1 and one_gpu:
        dist.init_process_group("gloo")

        def _host_allreduce(words):
            t = torch.from_numpy(words.view(np.int64))  # u64 sums as wrapping int64 sums
            dist.all_reduce(t)

        D.select_library("test")  # the hook exists in the test build only (numbers meaningless anyway)
        D.dsi_set_host_allreduce(_host_allreduce)
    elif world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfgs, tick = workload(args.workload, D.dsi_min_lookahead)
    # the e2e loops' inputs live in pinned host memory (the contract's H2D "from pinned host memory")
    _pin = torch.empty(max(1, cfgs.nbytes), dtype=torch.uint8, pin_memory=True)
    cfgs_pinned = _pin.numpy()[:cfgs.nbytes].view(D.CONFIG_DTYPE)
    cfgs_pinned[:] = cfgs

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: int) -> int:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.int64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return int(t.item())

    def fresh_nccl_id():
        """A new NCCL unique id for each handle (an id serves one communicator): made on rank 0,
        broadcast to all ranks (every rank calls this in the same order)."""
        if world == 1 or one_gpu:
            return None
        obj = [D.dsi_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    base_kw = dict(tick=tick, seed=W.SEED, device=local, rank=rank, world=world)
    kw = dict(base_kw, nccl_id=fresh_nccl_id())
    # one process per GPU: the results are gathered on rank 0 (DSI_F_REDUCE_TO_ROOT), so the
    # other ranks do not each copy back and finalize all n_cfg results on the shared host cores
    root = D.DSI_F_REDUCE_TO_ROOT if world > 1 else 0

    t_create = time.perf_counter()
    sim = D.Simulator(cfgs, flags=D.DSI_F_TIMING | root, **kw)
    create_s = time.perf_counter() - t_create
    comm = sim.comm_info()
    if comm["nranks"] != world:
        raise SystemExit(f"bench.py: the library's communicator has {comm['nranks']} ranks, WORLD_SIZE is {world}")
    stream = torch.cuda.ExternalStream(sim.stream(), device=torch.device("cuda", local))
    # result buffers allocated (and their pages touched) once, outside the timed region
    res = np.empty(cfgs.size, D.RESULT_DTYPE)
    resc = np.empty(cfgs.size, D.RESULT_DTYPE)
    res.view(np.uint8).fill(0)
    resc.view(np.uint8).fill(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    for _ in range(args.warmup):
        sim.run()
        sim.reduce()

    step_ms, kernel_ms = [], []
    launches = 0
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            torch.cuda.synchronize()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            sim.run()
            sim.reduce(res)
            ev1.record(stream)
            ev1.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            kernel_ms.append(sim.kernel_ms())
            launches += sim.launches()
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    barrier()
    total_ms = max_over_ranks(sum(step_ms))
    kern_ms = max_over_ranks(statistics.mean(kernel_ms))
    launches = sum_over_ranks(launches)
    tt = trial_tokens(cfgs)
    value = tt * args.steps / (total_ms / 1000.0)

    # shared-stream mode: same configs, same API call, one Philox pass per
    # trial per group of configs drawing identical indicators; reported beside `value`
    # because it changes what a simulated trial-token costs.  Its sums must be bit-identical.
    crn = None
    crn_exchange = None
    if not args.no_shared_streams:
        simc = D.Simulator(cfgs, flags=D.DSI_F_TIMING | D.DSI_F_SHARED_STREAMS | root, nccl_id=fresh_nccl_id(),
                           **base_kw)
        streamc = torch.cuda.ExternalStream(simc.stream(), device=torch.device("cuda", local))
        for _ in range(args.warmup):
            simc.run()
            simc.reduce(resc)
        barrier()
        torch.cuda.synchronize()
        c_ms, c_kern = [], []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(streamc)
            simc.run()
            simc.reduce_device()  # the exchange + partition check; the moments stay in HBM
            ev1.record(streamc)
            ev1.synchronize()
            c_ms.append(ev0.elapsed_time(ev1))
            c_kern.append(simc.kernel_ms())
        barrier()
        c_total = max_over_ranks(sum(c_ms))
        if rank == 0:
            simc.fetch(0, cfgs.size, resc)
        same = all(np.array_equal(resc[f], res[f]) for f in
                   ("sum_si_ticks", "sum_dsi_ticks", "sumsq_si_ticks", "sumsq_dsi_ticks", "sum_segments",
                    "n_dsi_gt_nonsi", "n_dsi_gt_si", "trials"))
        crn = {"value": tt * args.steps / (c_total / 1000.0), "unit": UNIT,
               "step": "dsi_sim_run + dsi_sim_reduce_device (CUDA events)",
               "ms_per_step": c_total / args.steps, "kernel_ms": max_over_ranks(statistics.mean(c_kern)),
               "launches_per_step": simc.launches(), "bit_identical_to_value_run": bool(same),
               "note": "DSI_F_SHARED_STREAMS: configs with equal (stream_id, floor(a 2^32), N, T) share "
                       "one Philox pass per trial; per-config results identical to the default mode"}
        heat_shared_s, cells_shared = heatmap_grid_times(simc, flush, args.steps)
        crn["e2e"], crn["e2e_all_results"] = fast_mode_e2e(simc, cfgs_pinned, resc, tt, args.steps, barrier,
                                                           max_over_ranks)
        crn_exchange = simc.comm_info()["heatmap_exchange"]
        simc.close()

    # means-only mode (DSI_F_MEANS_ONLY): segment-length histograms per indicator group,
    # per-config sums by linearity -- sums, means and heatmap cells identical to the value run
    means = None
    heat_means_s = None
    if not args.no_means:
        resm = np.zeros(cfgs.size, D.RESULT_DTYPE)
        simm = D.Simulator(cfgs, flags=D.DSI_F_TIMING | D.DSI_F_MEANS_ONLY | root, nccl_id=fresh_nccl_id(),
                           **base_kw)
        streamm = torch.cuda.ExternalStream(simm.stream(), device=torch.device("cuda", local))
        for _ in range(args.warmup):
            simm.run()
            simm.reduce(resm)
        barrier()
        torch.cuda.synchronize()
        m_ms, m_kern = [], []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(streamm)
            simm.run()
            simm.reduce_device()
            ev1.record(streamm)
            ev1.synchronize()
            m_ms.append(ev0.elapsed_time(ev1))
            m_kern.append(simm.kernel_ms())
        barrier()
        m_total = max_over_ranks(sum(m_ms))
        if rank == 0:
            simm.fetch(0, cfgs.size, resm)
        same = all(np.array_equal(resm[f], res[f]) for f in
                   ("sum_si_ticks", "sum_dsi_ticks", "sum_segments", "sum_si_iters", "trials",
                    "mean_si", "mean_dsi"))
        heat_means_s, cells_means = heatmap_grid_times(simm, flush, args.steps)
        e2e_m, e2e_m_all = fast_mode_e2e(simm, cfgs_pinned, resm, tt, args.steps, barrier, max_over_ranks)
        means = {"value": tt * args.steps / (m_total / 1000.0), "unit": UNIT,
                 "ms_per_step": m_total / args.steps, "kernel_ms": max_over_ranks(statistics.mean(m_kern)),
                 "launches_per_step": simm.launches(), "sums_and_means_identical_to_value_run": bool(same),
                 "e2e": e2e_m, "e2e_all_results": e2e_m_all,
                 "note": "DSI_F_MEANS_ONLY: one pass per indicator group builds the segment-length "
                         "histogram H[g]; each config's sums = sum_g H[g] x segment cost (linearity over "
                         "segments), identical integers to the value run; no second moments or per-trial "
                         "counters. ms_per_step = dsi_sim_run + dsi_sim_reduce_device (all-reduce and "
                         "partition check; the exact moments stay in HBM, dsi_sim_fetch / dsi_sim_heatmap "
                         "read what is wanted)"}
        simm.close()

    # "heatmap grid time" (BASELINE metric): run + all-reduce + on-device
    # per-cell argmin over k + the four ratio panels + D2H of the cells, end to end on the
    # host clock (dsi_sim_heatmap), in both modes; the cells must equal the
    # host product (dsi_heatmap) over the default run's reduced results
    heat_s, cells = heatmap_grid_times(sim, flush, args.steps)
    grid_s = max_over_ranks(statistics.median(heat_s))
    grid_shared_s = max_over_ranks(statistics.median(heat_shared_s)) if crn is not None else None
    grid_means_s = max_over_ranks(statistics.median(heat_means_s)) if heat_means_s else None  # (collective)
    # the other DSI reading (R24) on the same workload, every mode (collective: all ranks)
    fresh = None
    if not args.no_fresh:
        fresh = fresh_verifier_block(D, cfgs, tick, base_kw, root, fresh_nccl_id, flush, args.steps,
                                     res if rank == 0 else None)
        for k in ("per_config_kernel_ms", "grid_time_shared_streams_s", "grid_time_means_only_s"):
            fresh[k] = max_over_ranks(fresh[k])
    heat = None
    if rank == 0:
        t0 = time.perf_counter()
        host_cells = D.dsi_heatmap(cfgs, res)
        host_product_s = time.perf_counter() - t0
        same_cells = cells_equal(cells, host_cells)
        if crn is not None:
            same_cells = same_cells and cells_equal(cells_shared, host_cells)
        if means is not None:
            same_cells = same_cells and cells_equal(cells_means, host_cells)
        i = int(np.nanargmax(cells["r_min_dsi"]))
        heat = {"cells": int(cells.size),
                "grid_time_s": grid_s,
                "grid_time_shared_streams_s": grid_shared_s,
                "grid_time_means_only_s": grid_means_s,
                "host_product_s": host_product_s,
                "device_cells_equal_host_product": bool(same_cells),
                "max_r_min_dsi": float(cells["r_min_dsi"][i]),
                "at": {"t_drafter": float(cells["t_drafter"][i]), "accept_rate": float(cells["accept_rate"][i]),
                       "si_lookahead": int(cells["si_lookahead"][i]),
                       "dsi_lookahead": int(cells["dsi_lookahead"][i])},
                "reading": "default: literal Alg. 1 (P:112-142) + App. D (P:392-401), R5/R6 -- the "
                           "`value` run's; fresh_verifier: R24 (Thm 2's proof, P:445). They differ only "
                           "where k t_d > t_t (DESIGN.md 2.1)",
                "figures": fig_summary(cfgs, res, cells),
                "fresh_verifier": fresh,
                "note": "grid time = dsi_sim_run + dsi_sim_heatmap (all-reduce, one warp per cell on "
                        "the device, D2H of 10100 cells), host wall clock, median of the timed steps; "
                        "per-config, shared-stream and means-only modes, cells compared with the host "
                        "product of the value run"}
    # e2e through the public API with host buffers: update (validate + pinned H2D of the
    # config table) + run + reduce (all-reduce + D2H of the moments + FP64 finalise)
    h2d, d2h = sim.io_bytes()
    sim.update(cfgs_pinned)
    sim.run()
    sim.reduce()
    barrier()
    torch.cuda.synchronize()
    e2e_s = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        sim.update(cfgs_pinned)
        sim.run()
        sim.reduce(res)
        e2e_s.append(time.perf_counter() - t0)
    barrier()
    e2e_total = max_over_ranks(sum(e2e_s))
    e2e_value = tt * args.steps / e2e_total

    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak_instr = SM_COUNT * LANES_PER_SM_CLK * sm_max * 1e6  # thread-instr/s per GPU
    # dominant kernel = the trial kernel; algorithmic instructions of this rank's share
    achieved = alg_instructions(cfgs) / world / (kern_ms / 1000.0)
    mults = alg_multiplies(cfgs) / world  # this rank's share
    executed_wide = mults * 16.0 / 20.0    # rounds 2-9 of each call
    clk = clocks.summary()
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", "latest_ncu_summary.json")) as f:
            prof = json.load(f)
    except OSError:
        pass
    traffic = prof.get("dram_bytes_per_launch") if prof.get("workload") == args.workload else None
    ncu = None  # the pipe and issue utilisation ncu measured for this kernel (north_star: >= 60% issue)
    sf = None
    if prof.get("workload") == args.workload:
        sf = prof.get("set_full") or prof.get("set_full_stride20")
    if sf:
        def _pct(key):
            v = sf.get(key)
            return float(v[1]) if v else None
        ncu = {"issue_active_pct": _pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
               "fmaheavy_pct": _pct("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
               "alu_pct": _pct("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
               "source": f"profiles/{prof.get('round', '?')}_ncu_summary.json (--set full, "
                         + ("a full bench launch)" if prof.get("set_full") else "1/20 of the grid)")}

    multi = None
    if rank == 0 and not args.no_multi:
        multi = multi_drafter_block(args.steps, sm_max)
    barrier()

    # BASELINE configs[1], [3], [4] (cfg2, cfg4, cfg5: the large Monte Carlo) on the same GPUs
    others = None
    if not args.no_others and args.workload == "cfg3":
        others = other_workloads_block(D, ("cfg5", "cfg4", "cfg2"), args, base_kw, root, fresh_nccl_id, flush,
                                       barrier, max_over_ranks, world)

    halves = None
    if not args.no_halves:
        halves = rng_halves_block(D, cfgs, cfgs_pinned, tick, args, base_kw, root, fresh_nccl_id, flush, barrier,
                                  max_over_ranks, world, peak_instr)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle as O
        O.build()
        cpu = run_oracle_sample(cfgs, tick, args.cpu_seconds / 2, host_cores())
        one = run_oracle_sample(cfgs, tick, args.cpu_seconds / 2, 1)
        cpu["single_core"] = {"value": one["value"], "cores": 1, "sample": one["sample"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32/int64", "data": "synthetic",
            "config": {"workload": args.workload, "desc": WORKLOAD_DESC[args.workload],
                       "configs": int(cfgs.size), "trials": int(cfgs["n_trials"].sum()),
                       "trial_tokens_per_step": tt, "tick": tick, "seed": W.SEED,
                       "l2": "flushed between timed steps (256 MiB memset)", "parallelism": f"dp{world}",
                       "rng_layout": "one 32-bit Philox word per position (SURVEY 0.1(9), DESIGN R14); the "
                                     "halves layout (R26) is the rng_halves block"},
            # SURVEY 8(d).4's accounting: 11 + 10(1-a) algorithmic thread-instructions per
            # trial-token against the issue peak (148 SM x 4 SMSP x 32 lanes x clock); the
            # fmaheavy pipe that binds in ncu (Philox's IMAD.WIDE at a measured 4.1 cycles per
            # warp instruction) is the "fmaheavy" sub-object
            "roofline": {"bound": "alu", "achieved": achieved / 1e9, "peak": peak_instr / 1e9,
                         "unit": "Ginstr/s", "frac": achieved / peak_instr, "traffic": traffic,
                         "kernel": "dsi_trial_kernel", "kernel_ms": kern_ms,
                         "kernel_share_of_step": kern_ms / (total_ms / args.steps),
                         "work": "11 + 10(1-a) thread-instructions per trial-token (SURVEY 8(d).4): 10 for "
                                 "Philox4x32-10 (10 rounds x (2 mul-wide + 2 xor) / 4 words), 1 Bernoulli "
                                 "compare, 10 per rejection (segment walk + SI/DSI cost); per launch "
                                 f"{alg_instructions(cfgs) / world:.4e} instructions",
                         "peak_source": f"issue: 148 SM x 4 SMSP x 32 lanes x sm_max_mhz {sm_max:.0f} "
                                        "(MEASURED_PEAKS.json), one warp-instruction per SMSP per clock",
                         "frac_at_measured_clock": (achieved / (peak_instr * clk["sm_mhz"] / sm_max)
                                                    if clk.get("sm_mhz") else None),
                         # what a launch must move: the config table (112 B), the unit prefix (8 B) and
                         # the moment accumulators read and written by the L2 atomics (2 x 64 B)
                         "algorithmic_bytes": int(cfgs.size) * (112 + 8 + 2 * 64),
                         "ncu": ncu,
                         "fmaheavy": {
                             "achieved": executed_wide / (kern_ms / 1000.0) / 1e9,
                             "peak": mul_peak(sm_max) / 1e9, "unit": "G IMAD.WIDE/s",
                             "frac": executed_wide / (kern_ms / 1000.0) / mul_peak(sm_max),
                             "work": "the 32x32->64 multiplies the kernel must issue: Philox4x32-10 rounds "
                                     "2-9 (rounds 0-1 hoisted, DESIGN.md 6.1), 16 per call of 4 indicators, "
                                     "ceil((N-1)/4) calls per trial, configs with 0 < a < 1",
                             "peak_source": f"148 SM x 4 SMSP x 32 lanes / {imad_wide_cycles():.2f} cycles per "
                                            "warp IMAD.WIDE (profiles/r02_pipe_peaks.jsonl) x sm_max_mhz",
                             "trial_tokens_ceiling": _imad_ceiling(sm_max),
                             "trial_tokens_frac": (tt / world / (kern_ms / 1000.0)) / _imad_ceiling(sm_max)},
                         "multiplies_defined": {
                             "achieved": mults / (kern_ms / 1000.0) / 1e9, "peak": mul_peak(sm_max) / 1e9,
                             "unit": "Gmul/s", "frac": mults / (kern_ms / 1000.0) / mul_peak(sm_max),
                             "work": "all 20 multiplies per call Philox4x32-10 defines (a normalised speed, "
                                     "not a pipe utilisation: 4 of them are hoisted)"}},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches,
            "comm": dict(sim.comm_info(), shared_streams_heatmap_exchange=crn_exchange),
            "heatmap": heat,
            "shared_streams": crn,
            "means_only": means,
            "multi_drafter": multi,
            "other_workloads": others,
            "rng_halves": halves,
            "clocks": clk,
            "create_s": create_s,
            "wall_s_timed": wall,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--reference-seconds", type=float, default=90.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shared-streams", action="store_true")
    ap.add_argument("--no-multi", action="store_true", help="skip the multi-drafter block")
    ap.add_argument("--no-means", action="store_true", help="skip the means-only block")
    ap.add_argument("--no-fresh", action="store_true", help="skip the fresh-verifier (R24) heatmap block")
    ap.add_argument("--no-others", action="store_true", help="skip BASELINE's other configs (cfg5, cfg4, cfg2)")
    ap.add_argument("--no-halves", action="store_true", help="skip the DSI_F_RNG_HALVES block")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return relaunch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: launch one process per GPU "
                         f"(torch.distributed.run --nproc-per-node {args.gpus}) or drop the torchrun wrapper")
    if args.impl == "reference":
        return reference_arm(args)
    return ours(args)


def relaunch_command(gpus: int, argv, port: int) -> list:
    """torch.distributed.run command that runs this script on `gpus` processes of one node, as
    the driver launches it (the same flags)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def relaunch(gpus: int) -> int:
    """--gpus N > 1 outside torchrun: one process per GPU under torch.distributed.run (rank 0
    prints the line).  NCCL_DEBUG=INFO (INIT) makes each communicator's size visible in stderr."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = relaunch_command(gpus, sys.argv[1:], port)
    sys.stdout.flush()
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    sys.exit(main())

"""Command-line front end of the simulator (every number comes from libdsi_sim.so).

    python -m paper_2405_14105_b200 plan --t-target 1.0 --t-drafter 0.05 --sp 4
    python -m paper_2405_14105_b200 simulate --t-target 20.6 --t-drafter 6.8 --accept 0.93 \
        --lookahead 5 --sp 7 --n-tokens 50 --trials 100000 --tick 0.1
    python -m paper_2405_14105_b200 table2 [--trials 100000] [--sp 8] [--n-tokens 100]
    python -m paper_2405_14105_b200 heatmap [--trials 10000] [--k-max 200 | --k 5] [--csv out.csv] [--shared|--means] [--fresh]
    python -m paper_2405_14105_b200 multi --t-target 1.0 --drafter 0.02:0.5 --drafter 0.1:0.8 \
        --n-tokens 100 [--trials 100000]

`plan` is Eq. 1; `table2` evaluates the Table 2 (target, drafter, acceptance)
rows offline with lookahead in {1, 5, 10}, SI over all of them and DSI over the
Eq.-1-feasible ones (the protocol of P:273); `heatmap` is Fig. 3;
`multi` is Algorithm 1 with several drafters (latency:acceptance, fastest first), lookahead 1.
`heatmap` also runs sharded over GPUs under torchrun (one process per GPU; rank 0 writes the CSV):
    python -m torch.distributed.run --nproc-per-node 8 -m paper_2405_14105_b200 heatmap --means --csv h.csv
Exit codes: 0 success, 2 invalid arguments (DSI_E_RANGE / DSI_E_TICK / ...), 3 device error.
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from . import dsi_sim as D
from . import workloads as W


class UsageError(Exception):
    """Invalid arguments (exit code 2)."""


def cmd_plan(a) -> dict:
    """Eq. 1, every number from the library: latencies in whole ticks
    (R15, dsi_ticks), Assumption 2 (t_drafter <= t_target), SP >= 1."""
    tt, td = D.dsi_ticks(a.t_target, a.tick), D.dsi_ticks(a.t_drafter, a.tick)
    if td > tt:
        raise UsageError("t_drafter must not exceed t_target (Assumption 2)")
    if a.sp < 1:
        raise UsageError("sp must be >= 1")
    k = D.dsi_min_lookahead(tt, td, a.sp)
    procs = D.dsi_required_processors(tt, td, k)
    # beyond ceil(t_t / t_d) target servers (the k = 1 requirement) no lookahead needs more
    max_sp = D.dsi_required_processors(tt, td, 1) - 1
    feasible = D.dsi_eq1_feasible(tt, td, k, a.sp)
    if min(k, procs, max_sp, feasible) < 0:
        raise UsageError("invalid planner arguments")
    return {"min_lookahead": k, "processors": procs, "max_useful_sp": max_sp, "eq1_feasible_at_k": bool(feasible)}


def cmd_simulate(a) -> dict:
    cfg = np.zeros(1, D.CONFIG_DTYPE)
    cfg[0] = (a.t_target, a.t_drafter, a.accept, a.lookahead, a.sp, a.n_tokens, a.stream, a.trials,
              a.ttft_target, a.ttft_drafter)
    flags = (D.DSI_F_FRESH_VERIFIER if a.fresh else 0) | (D.DSI_F_RNG_HALVES if a.rng_halves else 0)
    with D.Simulator(cfg, tick=a.tick, seed=a.seed, flags=flags) as sim:
        r = sim.run().reduce()[0]
    return {k: (float(r[k]) if r.dtype[k].kind == "f" else int(r[k])) for k in r.dtype.names}


def table2(trials: int, sp: int, n_tokens: int, seed: int = W.SEED, device: int = 0,
           prefill: bool = False) -> list:
    """prefill: first forwards cost TTFT = Table-3 ratio x TPOT (P:273 'including prefilling')."""
    if prefill:
        cfgs, tick = W.cfg2_ttft(trials=trials, sp=sp, n_tokens=n_tokens)
    else:
        cfgs, tick = W.cfg2(trials=trials, sp=sp, n_tokens=n_tokens)
    with D.Simulator(cfgs, tick=tick, seed=seed, device=device) as sim:
        cells = sim.run().heatmap()  # on-device argmin over k (dsi_sim_heatmap)
    rows = []
    for (name, *_), c in zip(W.TABLE2_ROWS, cells):
        rows.append({"pair": name, "si_ms": float(c["si"]), "si_lookahead": int(c["si_lookahead"]),
                     "dsi_ms": float(c["dsi"]), "dsi_lookahead": int(c["dsi_lookahead"]),
                     "nonsi_ms": float(c["nonsi"]), "speedup_dsi_vs_si": float(c["r_si_dsi"])})
    return rows


def cmd_table2(a) -> list:
    """--sp / --n-tokens default to the protocol's own values: SP 8, N 100 (BASELINE configs[1])
    without --prefill; SP 7, N 50 with it."""
    sp = a.sp if a.sp is not None else (7 if a.prefill else 8)
    n = a.n_tokens if a.n_tokens is not None else (50 if a.prefill else 100)
    return table2(a.trials, sp, n, a.seed, prefill=a.prefill)


def _distributed_kw():
    """Under torchrun (WORLD_SIZE > 1): one process per GPU, a torch.distributed process group for
    the plumbing and a fresh NCCL unique id for the library's communicator.  DSI_BENCH_ONE_GPU=1
    (tests) keeps every rank on GPU 0 with gloo and the library's host all-reduce hook."""
    import os
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1:
        return {}, 0
    import torch
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("DSI_BENCH_ONE_GPU") == "1":
        local = 0
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
        D.select_library("test")  # the host all-reduce hook exists in the test build only
        D.dsi_set_host_allreduce(lambda w: dist.all_reduce(torch.from_numpy(w.view(np.int64))))
        return dict(device=local, rank=rank, world=world), rank
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [D.dsi_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return dict(device=local, rank=rank, world=world, nccl_id=obj[0]), rank


def cmd_heatmap(a) -> dict:
    if a.k:  # one lookahead for SI and DSI: the static panels of Fig. 5
        cfgs, tick = W.cfg3(trials=a.trials, k_min=a.k, k_max=a.k, sp=a.sp, n_tokens=a.n_tokens)
    else:
        cfgs, tick = W.cfg3(trials=a.trials, k_max=a.k_max, sp=a.sp, n_tokens=a.n_tokens)
    flags = ((D.DSI_F_SHARED_STREAMS if a.shared else 0) | (D.DSI_F_FRESH_VERIFIER if a.fresh else 0) |
             (D.DSI_F_MEANS_ONLY if a.means else 0) | (D.DSI_F_RNG_HALVES if a.rng_halves else 0))
    kw, rank = _distributed_kw()  # torchrun: the grid is sharded over the ranks' GPUs
    with D.Simulator(cfgs, tick=tick, seed=a.seed, flags=flags, **kw) as sim:
        cells = sim.run().heatmap()  # collective: every rank gets every cell
    if a.csv and rank == 0:
        D.dsi_heatmap_csv(cells, a.csv)
    i = int(np.nanargmax(cells["r_min_dsi"]))
    return {"cells": int(cells.size), "csv": a.csv,
            "max_min_si_nonsi_over_dsi": float(cells["r_min_dsi"][i]),
            "at": {"t_drafter": float(cells["t_drafter"][i]), "accept_rate": float(cells["accept_rate"][i])},
            "si_slower_than_nonsi_cells": int(np.sum(cells["r_nonsi_si"] < 1.0)),
            "dsi_slower_than_si_cells": int(np.sum(cells["r_si_dsi"] < 1.0))}


def cmd_multi(a) -> dict:
    ds = []
    for d in a.drafter:
        t, _, acc = d.partition(":")
        ds.append((float(t), float(acc)))
    cfg = W.multi_rows([(a.t_target, tuple(t for t, _ in ds), tuple(x for _, x in ds))], a.trials, a.n_tokens,
                       a.stream)
    r = D.dsi_multi_simulate(cfg, tick=a.tick, seed=a.seed, flags=D.DSI_F_MEANS_ONLY if a.means else 0)[0][0]
    m = len(ds) + 1
    return {"models": m, "mean_dsi": float(r["mean_dsi"]), "std_dsi": float(r["std_dsi"]),
            "mean_nonsi": float(r["mean_nonsi"]), "speedup_vs_nonsi": float(r["mean_nonsi"] / r["mean_dsi"]),
            "settled_share": [float(x) / (int(r["trials"]) * max(a.n_tokens - 1, 1)) for x in r["sum_settled"][:m]],
            "n_dsi_gt_nonsi": int(r["n_dsi_gt_nonsi"]), "trials": int(r["trials"])}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2405_14105_b200")
    ap.add_argument("--seed", type=int, default=W.SEED)
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("plan", help="Eq. 1: minimal lookahead and processors")
    p.add_argument("--t-target", type=float, required=True)
    p.add_argument("--t-drafter", type=float, required=True)
    p.add_argument("--sp", type=int, required=True)
    p.add_argument("--tick", type=float, default=0.01)
    p = sub.add_parser("simulate", help="one configuration")
    for f in ("--t-target", "--t-drafter", "--accept"):
        p.add_argument(f, type=float, required=True)
    for f in ("--lookahead", "--sp", "--n-tokens"):
        p.add_argument(f, type=int, required=True)
    p.add_argument("--trials", type=int, default=100_000)
    p.add_argument("--tick", type=float, default=0.01)
    p.add_argument("--stream", type=int, default=0)
    p.add_argument("--ttft-target", type=float, default=0.0, help="first target forward (0 = TPOT)")
    p.add_argument("--ttft-drafter", type=float, default=0.0, help="first drafter forward (0 = TPOT)")
    p.add_argument("--fresh", action="store_true", help="DSI_F_FRESH_VERIFIER (DESIGN.md R24)")
    p.add_argument("--rng-halves", action="store_true", help="DSI_F_RNG_HALVES (DESIGN.md R26)")
    p = sub.add_parser("table2", help="Table 2 pairs offline, lookahead in {1, 5, 10}")
    p.add_argument("--trials", type=int, default=100_000)
    p.add_argument("--sp", type=int, default=None, help="default 8, or 7 with --prefill (P:273)")
    p.add_argument("--n-tokens", type=int, default=None, help="default 100, or 50 with --prefill (P:273)")
    p.add_argument("--prefill", action="store_true",
                   help="TTFT = Table-3 ratio x TPOT for each model's first forward (use --trials <= 1e4)")
    p = sub.add_parser("heatmap", help="Fig. 3 grid; optional CSV")
    p.add_argument("--trials", type=int, default=10_000)
    p.add_argument("--k-max", type=int, default=200)
    p.add_argument("--k", type=int, default=0, help="a single lookahead (Fig. 5 uses 5; with --fresh)")
    p.add_argument("--sp", type=int, default=7)
    p.add_argument("--n-tokens", type=int, default=100)
    p.add_argument("--csv", default=None)
    p.add_argument("--shared", action="store_true", help="DSI_F_SHARED_STREAMS")
    p.add_argument("--means", action="store_true", help="DSI_F_MEANS_ONLY (segment histograms; no std)")
    p.add_argument("--fresh", action="store_true", help="DSI_F_FRESH_VERIFIER (DESIGN.md R24)")
    p.add_argument("--rng-halves", action="store_true", help="DSI_F_RNG_HALVES (DESIGN.md R26)")
    p = sub.add_parser("multi", help="Alg. 1 with several drafters (lookahead 1, unbounded threads)")
    p.add_argument("--t-target", type=float, required=True)
    p.add_argument("--drafter", action="append", required=True, help="latency:acceptance, fastest first")
    p.add_argument("--n-tokens", type=int, required=True)
    p.add_argument("--trials", type=int, default=100_000)
    p.add_argument("--tick", type=float, default=0.01)
    p.add_argument("--stream", type=int, default=0)
    p.add_argument("--means", action="store_true", help="DSI_F_MEANS_ONLY (no std)")
    a = ap.parse_args(argv)
    try:
        out = {"plan": cmd_plan, "simulate": cmd_simulate, "table2": cmd_table2, "heatmap": cmd_heatmap,
               "multi": cmd_multi}[a.cmd](a)
    except UsageError as e:
        print(str(e), file=sys.stderr)
        return 2
    except D.DsiError as e:
        print(str(e), file=sys.stderr)
        return 3 if e.status in (D.DSI_E_DEVICE, D.DSI_E_COMM, D.DSI_E_NOMEM) else 2
    import os
    if os.environ.get("RANK", "0") == "0":  # under torchrun only rank 0 reports
        print(json.dumps(out, indent=1))
    return 0

"""World-size-2 gloo test of the multi-GPU host logic on CPU.

Each rank takes its contiguous, cost-balanced share of the (config, trial-block) units
from the library's sharder (dsi_shard_bounds), simulates it (here with the CPU oracle,
the only simulator a CPU box can run), and the per-config integer moments are summed
with one all_reduce — the same exchange dsi_sim_reduce performs with NCCL.  The sums
must equal a single-process run bit for bit, for several partitions.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2405_14105_b200 import dsi_sim as D
from paper_2405_14105_b200 import workloads as W

FIELDS = ("sum_acc", "sum_m", "sum_iters", "sum_si", "sum_dsi", "sumsq_si", "sumsq_dsi",
          "n_dsi_gt_nonsi", "n_dsi_gt_si", "trials")
BLOCK = 37  # trials per unit (deliberately not a divisor of T)


def _configs():
    cfgs, tick = W.fuzz(12, seed=17, trials=150)
    return cfgs, tick


def _units(cfgs):
    units = []  # (config index, first trial, count)
    for c, row in enumerate(cfgs):
        T = int(row["n_trials"])
        for f in range(0, T, BLOCK):
            units.append((c, f, min(BLOCK, T - f)))
    cost = np.array([n * int(cfgs[c]["n_tokens"]) * (11 + 10 * (1 - float(cfgs[c]["accept_rate"])))
                     for c, _, n in units])
    return units, cost


def _simulate(cfgs, tick, units):
    acc = np.zeros((cfgs.size, len(FIELDS)), np.int64)
    for c, first, n in units:
        row = cfgs[c]
        oc = O.Config(O.ticks(float(row["t_target"]), tick), O.ticks(float(row["t_drafter"]), tick),
                      float(row["accept_rate"]), int(row["lookahead"]), int(row["sp_degree"]),
                      int(row["n_tokens"]), int(row["stream_id"]))
        r = O.run(oc, W.SEED, first, n, per_trial=False)
        acc[c] += np.array([np.int64(np.uint64(r[f]).astype(np.int64)) for f in FIELDS])
    return acc


def _worker(rank, world, port, parts, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfgs, tick = _configs()
    units, cost = _units(cfgs)
    bounds = D.dsi_shard_bounds(cost, parts)
    mine = []
    for p in range(rank, parts, world):  # each rank owns parts p = rank, rank+world, ...
        mine += units[int(bounds[p]):int(bounds[p + 1])]
    acc = torch.from_numpy(_simulate(cfgs, tick, mine))
    dist.all_reduce(acc, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put(acc.numpy().tobytes())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("parts", [2, 5])
def test_two_rank_partition_allreduce_is_bit_identical(parts):
    cfgs, tick = _configs()
    units, _ = _units(cfgs)
    want = _simulate(cfgs, tick, units)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()  # both ranks rendezvous on it
    procs = [ctx.Process(target=_worker, args=(r, 2, port, parts, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=300), dtype=np.int64).reshape(want.shape)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got, want)


def test_sharder_balances_cost():
    cfgs, _ = W.cfg3(k_max=5, trials=1000, cells=slice(None, None, 50))
    units = []
    for c, row in enumerate(cfgs):
        for f in range(0, int(row["n_trials"]), 128):
            units.append((c, f, min(128, int(row["n_trials"]) - f)))
    cost = np.array([n * 100 * (11 + 10 * (1 - float(cfgs[c]["accept_rate"]))) for c, _, n in units])
    for parts in (2, 4, 8):
        b = D.dsi_shard_bounds(cost, parts)
        shares = np.array([cost[b[j]:b[j + 1]].sum() for j in range(parts)])
        assert shares.max() / shares.mean() < 1.01


# ---- multi-drafter DSI (dsi_multi_simulate's world > 1 path): the same exchange --------------
MULTI_BLOCK = 29


def _multi_units(cfgs):
    units = []
    for c, row in enumerate(cfgs):
        for f in range(0, int(row["n_trials"]), MULTI_BLOCK):
            units.append((c, f, min(MULTI_BLOCK, int(row["n_trials"]) - f)))
    cost = np.array([n * (1.0 + int(cfgs[c]["n_tokens"])) for c, _, n in units], dtype=np.float64)
    return units, cost


def _multi_simulate(cfgs, tick, units):
    acc = np.zeros((cfgs.size, 3 + O.MAX_MODELS), np.int64)
    for c, first, n in units:
        row = cfgs[c]
        nd = int(row["n_drafters"])
        oc = O.MultiConfig(O.ticks(float(row["t_target"]), tick),
                           tuple(O.ticks(float(x), tick) for x in row["t_drafter"][:nd]),
                           tuple(float(x) for x in row["accept_rate"][:nd]), int(row["n_tokens"]),
                           int(row["stream_id"]))
        r = O.multi_run(oc, W.SEED, first, n, per_trial=False)
        acc[c, 0] += r["trials"]
        acc[c, 1] += r["sum_dsi"]
        acc[c, 2] += np.uint64(r["sumsq_dsi"]).astype(np.int64)
        acc[c, 3:3 + len(r["sum_settled"])] += r["sum_settled"]
    return acc


def _multi_worker(rank, world, port, parts, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfgs, tick = W.multi_fuzz(10, seed=31, n_max=50, trials=120)
    units, cost = _multi_units(cfgs)
    bounds = D.dsi_shard_bounds(cost, parts)
    per = parts // world  # contiguous parts per rank, as dsi_multi_simulate assigns them
    mine = []
    for p in range(rank * per, (rank + 1) * per):
        mine += units[int(bounds[p]):int(bounds[p + 1])]
    acc = torch.from_numpy(_multi_simulate(cfgs, tick, mine))
    dist.all_reduce(acc, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put(acc.numpy().tobytes())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("parts", [2, 6])
def test_two_rank_multi_drafter_partition_allreduce_is_bit_identical(parts):
    cfgs, tick = W.multi_fuzz(10, seed=31, n_max=50, trials=120)
    units, _ = _multi_units(cfgs)
    want = _multi_simulate(cfgs, tick, units)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_multi_worker, args=(r, 2, port, parts, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=300), dtype=np.int64).reshape(want.shape)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got, want)

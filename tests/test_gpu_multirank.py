"""Two ranks on ONE GPU through the library's multi-rank paths (tests what a multi-GPU run does
except NCCL itself, which refuses two ranks on one GPU -- profiles/two_rank_one_gpu.py).

Each rank is a process with a gloo process group; the library's cross-rank sums go through the
host all-reduce hook (dsi_set_host_allreduce) instead of NCCL.  Everything else is the multi-rank
code: the cost-balanced partition of units across ranks, the all-reduce of moments / histograms /
heatmap cells, DSI_F_REDUCE_TO_ROOT, the cell-aligned means-only heatmap, the multi-drafter call.
Rank 0's results must equal a single-process run bit for bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

D = pytest.importorskip("paper_2405_14105_b200.dsi_sim")
from paper_2405_14105_b200 import workloads as W  # noqa: E402

SEED = W.SEED


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cases():
    fz, ftick = W.fuzz(30, seed=13, trials=700)
    c3, tick3 = W.cfg3(trials=600, k_max=20, cells=slice(3, 10100, 151))
    ttft, ttick = W.cfg2_ttft(trials=500)
    return [("default", fz, ftick, 0), ("root", fz, ftick, D.DSI_F_REDUCE_TO_ROOT),
            ("hist", fz, ftick, D.DSI_F_HIST), ("shared", c3, tick3, D.DSI_F_SHARED_STREAMS),
            ("means", c3, tick3, D.DSI_F_MEANS_ONLY), ("means_ttft", ttft, ttick, D.DSI_F_MEANS_ONLY),
            ("fresh", fz, ftick, D.DSI_F_FRESH_VERIFIER),
            ("shared_fresh", c3, tick3, D.DSI_F_SHARED_STREAMS | D.DSI_F_FRESH_VERIFIER),
            ("shared_ttft", ttft, ttick, D.DSI_F_SHARED_STREAMS),
            ("halves", fz, ftick, D.DSI_F_RNG_HALVES),
            ("halves_shared", c3, tick3, D.DSI_F_SHARED_STREAMS | D.DSI_F_RNG_HALVES),
            ("halves_means", c3, tick3, D.DSI_F_MEANS_ONLY | D.DSI_F_RNG_HALVES)]


CURRENT = {"case": None}


def _run_all(rank, world):
    out = {}
    for name, cfgs, tick, flags in _cases():
        CURRENT["case"] = name
        with D.Simulator(cfgs, tick=tick, seed=SEED, flags=flags, rank=rank, world=world) as sim:
            sim.run()
            res = sim.reduce()  # collective: every rank calls it (with REDUCE_TO_ROOT only rank 0's is filled)
            cells = sim.heatmap()
            hist = sim.hist(1) if flags & D.DSI_F_HIST else None
            # the heatmap's own exchange (cells, or the moments first) with no reduce before it, the
            # deferred reduce, and an update (device path where eligible) of the drafter latencies
            cells_first = sim.run().heatmap()
            if not flags & D.DSI_F_HIST:
                sim.run().reduce_device()
                fetched = sim.fetch() if rank == 0 or not flags & D.DSI_F_REDUCE_TO_ROOT else None
                new = cfgs.copy()
                # (a new shared-stream plan may change the unit count, and a TTFT config may stop being
                # one: both need a new handle by contract)
                if not flags & D.DSI_F_SHARED_STREAMS and not np.any(cfgs["ttft_drafter"]):
                    new["t_drafter"] = np.minimum(new["t_target"], new["t_drafter"] + tick)
                upd = sim.update(new).run().reduce()
            else:
                fetched = upd = None
        out[name] = (res, cells, hist, cells_first, fetched if rank == 0 else None, upd)
    mc, mtick = W.multi_fuzz(15, seed=5, trials=900)
    out["multi"] = (D.dsi_multi_simulate(mc, tick=mtick, seed=SEED, rank=rank, world=world)[0], None, None)
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allreduce(words):
        if os.environ.get("DSI_DEBUG_AR"):
            print(f"rank {rank} case {CURRENT['case']} allreduce {words.size}", flush=True)
        t = torch.from_numpy(words.view(np.int64))  # u64 sums as wrapping int64 sums
        dist.all_reduce(t)

    D.select_library("test")  # the host all-reduce hook exists in the test build only
    D.dsi_set_host_allreduce(allreduce)
    try:
        res = _run_all(rank, world)
        q.put((rank, "ok", res if rank == 0 else None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e)))
    dist.barrier()
    dist.destroy_process_group()


def _same(a, b):
    if a is None or b is None:
        return a is None and b is None
    if isinstance(a, tuple):
        return all(_same(x, y) for x, y in zip(a, b))
    for f in a.dtype.names:
        x, y = np.asarray(a[f]), np.asarray(b[f])
        if x.dtype.kind == "f":
            if not (np.array_equal(np.isnan(x), np.isnan(y)) and np.array_equal(x[~np.isnan(x)], y[~np.isnan(y)])):
                return False
        elif not np.array_equal(x, y):
            return False
    return True


def test_two_ranks_on_one_gpu_equal_one_process():
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    want = _run_all(0, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        r, status, payload = q.get(timeout=600)
        assert status == "ok", payload
        got[r] = payload
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for name, w in want.items():
        g = got[0][name]
        assert _same(g[0], w[0]), name
        assert _same(g[1], w[1]), name
        if w[2] is not None:
            assert all(np.array_equal(x, y) for x, y in zip(g[2], w[2])), name
        for i, what in ((3, "cells (heatmap exchange only)"), (4, "fetch after reduce_device"), (5, "after update")):
            if i < len(w):
                assert _same(g[i], w[i]), (name, what)

"""Probe: can two processes on ONE GPU form an NCCL communicator through the library?
(NCCL normally refuses duplicate GPUs; this records what this box does.)"""
import multiprocessing as mp
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, nid, q):
    from paper_2405_14105_b200 import dsi_sim as D, workloads as W
    cfgs, tick = W.fuzz(20, seed=3, trials=200)
    try:
        with D.Simulator(cfgs, tick=tick, seed=W.SEED, rank=rank, world=2, nccl_id=nid) as sim:
            res = sim.run().reduce()
            q.put((rank, "ok", int(res["sum_dsi_ticks"].sum())))
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", str(e)[:300]))


if __name__ == "__main__":
    from paper_2405_14105_b200 import dsi_sim as D
    nid = D.dsi_nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, nid, q)) for r in range(2)]
    for p in ps:
        p.start()
    for _ in range(2):
        print(q.get(timeout=150), flush=True)
    for p in ps:
        p.join(timeout=30)

"""SURVEY 8(e)'s cell-aligned exchange: when the shards are snapped to heatmap-cell starts
(per-config mode) or group starts (shared-stream mode), dsi_sim_heatmap evaluates each part's
cells from its own moments and exchanges only the cells.  The cells must be bit-identical to
the one-shard run's (the all-reduce path), for any shard count -- on one GPU the shards run
back to back (n_shards); tests/test_gpu_multirank.py runs two ranks."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

D = pytest.importorskip("paper_2405_14105_b200.dsi_sim")
from paper_2405_14105_b200 import workloads as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def cells_same(a, b):
    for f in a.dtype.names:
        assert np.array_equal(a[f], b[f], equal_nan=a[f].dtype.kind == "f"), f


@pytest.mark.parametrize("flags", [0, D.DSI_F_SHARED_STREAMS, D.DSI_F_SHARED_STREAMS | D.DSI_F_FRESH_VERIFIER,
                                   D.DSI_F_MEANS_ONLY])
def test_cell_local_heatmap_equals_all_reduce_path(flags):
    # 25 drafter latencies x 101 acceptance rates x k 1..12: 101 groups of 300 configs
    cfgs, tick = W.cfg3(trials=1500, k_max=12, cells=slice(0, 2525))
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
        want = sim.run().heatmap()
        res = sim.reduce()
    for shards in (3, 8):
        with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags, n_shards=shards) as sim:
            got = sim.run().heatmap()
            assert sim.comm_info()["heatmap_exchange"] == "cells", shards
            cells_same(got, want)
            r2 = sim.reduce()
            for f in ("sum_si_ticks", "sum_dsi_ticks", "sum_segments", "trials"):
                assert np.array_equal(r2[f], res[f]), (shards, f)


def test_unsnappable_work_falls_back_to_the_all_reduce():
    """One config cannot be split into whole cells over 3 shards without losing the balance:
    the shards stay cost-balanced and the heatmap all-reduces the moments first."""
    cfgs, tick = W.cfg1(trials=60000)
    with D.Simulator(cfgs, tick=tick, seed=W.SEED) as sim:
        want = sim.run().heatmap()
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, n_shards=3) as sim:
        got = sim.run().heatmap()
        assert sim.comm_info()["heatmap_exchange"] == "moments"
        cells_same(got, want)

"""GPU tests of the deferred reduce (dsi_sim_reduce_device + dsi_sim_fetch): the exchange step
and the partition check run on the device, the exact moments stay in HBM, and any range of
results is derived on request -- bit-identical to dsi_sim_reduce's, which is bit-exact against
the oracle (tests/test_gpu_parity.py); a sample is also checked against the oracle directly."""
import numpy as np
import pytest

from helpers import assert_result_equals_oracle, oracle_sums

pytestmark = pytest.mark.gpu

D = pytest.importorskip("paper_2405_14105_b200.dsi_sim")
from paper_2405_14105_b200 import workloads as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def same(a, b):
    for f in a.dtype.names:
        x, y = a[f], b[f]
        if x.dtype.kind == "f":
            assert np.array_equal(x, y, equal_nan=True), f
        else:
            assert np.array_equal(x, y), f


def cells_same(a, b):
    for f in a.dtype.names:
        assert np.array_equal(a[f], b[f], equal_nan=a[f].dtype.kind == "f"), f


@pytest.mark.parametrize("flags", [0, D.DSI_F_SHARED_STREAMS, D.DSI_F_MEANS_ONLY, D.DSI_F_FRESH_VERIFIER])
def test_fetch_equals_reduce(flags):
    cfgs, tick = W.fuzz(120, seed=5, trials=700)
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
        want = sim.run().reduce()
        cells_want = sim.heatmap()
        sim.run().reduce_device()
        got = sim.fetch()
        same(got, want)
        for first, count in ((0, 1), (7, 33), (cfgs.size - 5, 5), (50, 0)):
            same(sim.fetch(first, count), want[first:first + count])
        cells_same(sim.heatmap(), cells_want)  # no second all-reduce after reduce_device


def test_fetch_against_the_oracle():
    cfgs, tick = W.cfg2(trials=2000)
    with D.Simulator(cfgs, tick=tick, seed=W.SEED) as sim:
        sim.run().reduce_device()
        got = sim.fetch(3, 6)
    for j in range(6):
        assert_result_equals_oracle(got[j], oracle_sums(cfgs[3 + j], tick, W.SEED), tick, ctx=j)


def test_call_order_and_ranges():
    cfgs, tick = W.fuzz(20, seed=2, trials=100)
    with D.Simulator(cfgs, tick=tick, seed=W.SEED) as sim:
        with pytest.raises(D.DsiError) as e:
            sim.reduce_device()
        assert e.value.status == D.DSI_E_STATE  # before run
        sim.run()
        with pytest.raises(D.DsiError) as e:
            sim.fetch(0, 1)
        assert e.value.status == D.DSI_E_STATE  # before a reduce
        sim.reduce_device()
        with pytest.raises(D.DsiError) as e:
            sim.fetch(15, 6)
        assert e.value.status == D.DSI_E_RANGE
        sim.run()
        with pytest.raises(D.DsiError) as e:
            sim.fetch(0, 1)
        assert e.value.status == D.DSI_E_STATE  # a new run invalidates the reduced moments
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=D.DSI_F_HIST) as sim:
        sim.run()
        with pytest.raises(D.DsiError) as e:
            sim.reduce_device()
        assert e.value.status == D.DSI_E_STATE


def test_nccl_one_rank():
    cfgs, tick = W.fuzz(40, seed=9, trials=300)
    with D.Simulator(cfgs, tick=tick, seed=W.SEED) as sim:
        want = sim.run().reduce()
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, rank=0, world=1, nccl_id=D.dsi_nccl_unique_id()) as sim:
        sim.run().reduce_device()
        same(sim.fetch(), want)

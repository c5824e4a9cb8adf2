"""The device path of dsi_sim_update (dsi_stage.cu): the new configurations are validated and
converted on the GPU with the host's own functions (dsi_convert.h) and committed when no plan
needs rebuilding; otherwise the host path runs.  Either way the handle must behave exactly like a
fresh handle created with the new configurations, report the host path's errors (status and
message) and keep its previous configurations when an update fails."""
import numpy as np
import pytest

from helpers import assert_result_equals_oracle, oracle_sums

pytestmark = pytest.mark.gpu

D = pytest.importorskip("paper_2405_14105_b200.dsi_sim")
from paper_2405_14105_b200 import workloads as W  # noqa: E402

SUMS = ("sum_dsi_ticks", "sum_si_ticks", "sumsq_dsi_ticks", "sumsq_si_ticks", "sum_segments", "sum_si_iters",
        "n_dsi_gt_nonsi", "n_dsi_gt_si", "trials", "mean_dsi", "mean_si", "eq1_feasible", "min_lookahead")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def fresh(cfgs, tick, flags):
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
        return sim.run().reduce(), sim.run().heatmap()


def same(a, b, ctx=""):
    for f in SUMS:
        assert np.array_equal(a[f], b[f], equal_nan=a[f].dtype.kind == "f"), (ctx, f)


def cells_same(a, b):
    for f in a.dtype.names:
        assert np.array_equal(a[f], b[f], equal_nan=a[f].dtype.kind == "f"), f


def grid():
    cfgs, tick = W.cfg3(trials=400, k_max=12, cells=slice(0, 404))  # 4 t_d x 101 a x k 1..12
    return cfgs, tick


def changed_latencies(cfgs):
    """New drafter latencies and lookaheads; N and the max lookahead unchanged."""
    new = cfgs.copy()
    new["t_drafter"] = np.round(new["t_drafter"] * 2 + 0.01, 2)
    new["lookahead"] = np.maximum(1, 13 - new["lookahead"])
    return new


def pinned_copy(cfgs):
    import torch
    buf = torch.empty(cfgs.nbytes, dtype=torch.uint8, pin_memory=True).numpy()
    view = buf.view(D.CONFIG_DTYPE)
    view[:] = cfgs
    return view, buf


@pytest.mark.parametrize("flags", [0, D.DSI_F_MEANS_ONLY, D.DSI_F_FRESH_VERIFIER, D.DSI_F_SHARED_STREAMS])
@pytest.mark.parametrize("pinned", [False, True])
def test_update_equals_a_fresh_handle(flags, pinned):
    cfgs, tick = grid()
    new = changed_latencies(cfgs)
    want, want_cells = fresh(new, tick, flags)
    src, keep = pinned_copy(new) if pinned else (new, None)
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
        sim.run().heatmap()
        for _ in range(2):  # the second update starts from a device-committed one
            sim.update(src)
            got = sim.run().reduce()
            same(got, want, ctx=(flags, pinned))
            cells_same(sim.run().heatmap(), want_cells)
        sim.update(cfgs)  # and back
        same(sim.run().reduce(), fresh(cfgs, tick, flags)[0], ctx="back")
    del keep


def test_identical_update_and_fetch_against_the_oracle():
    cfgs, tick = W.cfg2(trials=3000)
    src, keep = pinned_copy(cfgs)
    with D.Simulator(cfgs, tick=tick, seed=W.SEED) as sim:
        for _ in range(3):
            sim.update(src).run().reduce_device()
        got = sim.fetch(0, 5)
    for i in range(5):
        assert_result_equals_oracle(got[i], oracle_sums(cfgs[i], tick, W.SEED), tick, ctx=i)
    del keep


@pytest.mark.parametrize("flags", [0, D.DSI_F_MEANS_ONLY])
def test_errors_are_the_host_paths_and_nothing_changes(flags):
    cfgs, tick = grid()
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
        before = sim.run().reduce()
        sim.update(changed_latencies(cfgs))  # a device-committed state first
        mid = sim.run().reduce()
        for field, value, status, msg in (("t_drafter", 5.0, D.DSI_E_RANGE, "config 17: t_drafter > t_target"),
                                          ("t_target", 1.234567, D.DSI_E_TICK, "config 17: t_target is not"),
                                          ("n_trials", 401, D.DSI_E_RANGE, "config 17: n_trials")):
            bad = changed_latencies(cfgs)
            bad[field][17] = value
            bad[field][40] = value
            with pytest.raises(D.DsiError) as e:
                sim.update(bad)
            assert e.value.status == status and msg in str(e.value), (field, str(e.value))
            same(sim.run().reduce(), mid, ctx=field)  # the failed update changed nothing
        sim.update(cfgs)
        same(sim.run().reduce(), before, ctx="restored")


@pytest.mark.parametrize("flags", [0, D.DSI_F_MEANS_ONLY, D.DSI_F_FRESH_VERIFIER])
def test_random_update_sequence(flags):
    """A sequence of random updates -- valid ones (new latencies, lookaheads, SP, acceptance) and
    invalid ones (one field broken in one config) -- against fresh handles: every valid update
    gives the fresh handle's results, every invalid one create's status and message, and leaves
    the handle as it was."""
    rng = np.random.default_rng(99)
    cfgs, tick = W.fuzz(60, seed=21, trials=300)
    cfgs["ttft_target"] = 0.0
    cfgs["ttft_drafter"] = 0.0
    cur = cfgs.copy()
    with D.Simulator(cfgs, tick=tick, seed=W.SEED, flags=flags) as sim:
        sim.run().reduce()
        for step in range(10):
            new = cur.copy()
            if flags & D.DSI_F_MEANS_ONLY:  # (the groups: stream, a, N, T must stay)
                new["t_drafter"] = np.maximum(1.0, np.minimum(new["t_target"], new["t_drafter"] + rng.integers(-3, 4, new.size)))
                new["sp_degree"] = rng.integers(1, 9, new.size)
            else:
                new["accept_rate"] = np.round(rng.random(new.size), 2)
                new["lookahead"] = np.minimum(new["lookahead"], rng.integers(1, 13, new.size))
                new["t_drafter"] = np.maximum(1.0, np.minimum(new["t_target"], new["t_drafter"] + rng.integers(-3, 4, new.size)))
            if step % 3 == 2:  # break one config
                i = int(rng.integers(0, new.size))
                new["t_drafter"][i] = new["t_target"][i] + 1.0
                with pytest.raises(D.DsiError) as e:
                    sim.update(new)
                with pytest.raises(D.DsiError) as e2:
                    D.Simulator(new, tick=tick, seed=W.SEED, flags=flags)
                assert e.value.status == e2.value.status and str(e.value) == str(e2.value)
                same(sim.run().reduce(), fresh(cur, tick, flags)[0], ctx=("kept", step))
                continue
            sim.update(new)
            same(sim.run().reduce(), fresh(new, tick, flags)[0], ctx=("step", step))
            cur = new

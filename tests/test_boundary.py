"""CPU tests of the C-ABI library: it loads, exports every symbol include/dsi_sim.h
declares, and its host-only logic (validation, planner, sharder) behaves.  No compute
call is made without a GPU: on this box dsi_sim_create must stop with DSI_E_DEVICE
after validation passes."""
import json
import os
import random
import re

import numpy as np
import pytest

import oracle as O
from paper_2405_14105_b200 import dsi_sim as D
from paper_2405_14105_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dsi_sim.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dsi_[a-z_0-9]+)\s*\(", src)))


def test_every_header_symbol_is_exported_and_bound():
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(D.lib, n), n            # dlsym succeeds
        assert n in D.EXPORTED, n               # the binding declares it
        assert hasattr(D, n) or n in ("dsi_status_str", "dsi_sim_last_error",
                                      "dsi_last_create_error", "dsi_abi_version"), n


def test_test_hooks_only_in_the_test_builds():
    """include/dsi_sim_testing.h exists in libdsi_sim_test.so / _mutant.so only; the product
    exports none of it.  Every build embeds the SHA-256 of the current sources (build.py)."""
    from paper_2405_14105_b200 import build as B
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "dsi_sim_testing.h")).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(dsi_[a-z_0-9]+)\s*\(", src)))
    assert names == sorted(D.TEST_EXPORTED)
    prod, test = D.load_library("product"), D.load_library("test")
    for n in names:
        assert not hasattr(prod, n), n
        assert hasattr(test, n), n
    for variant in ("product", "test", "mutant"):
        assert not B.stale(variant), variant
    assert D.dsi_build_id() == B.build_id("product")


def test_abi_version_and_status_strings():
    assert D.lib.dsi_abi_version() == D.DSI_ABI_VERSION
    for s in range(10):
        assert D.lib.dsi_status_str(s).decode().startswith("DSI_")


def test_planner_matches_paper_examples():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "planner.json")))
    for e in g["min_lookahead"]:
        assert D.dsi_min_lookahead(e["t_target"], e["t_drafter"], e["sp"]) == e["k"], e["cite"]
    for e in g["required_processors"]:
        assert D.dsi_required_processors(e["t_target"], e["t_drafter"], e["k"]) == e["procs"], e["cite"]


def test_planner_matches_definition():
    """Eq. 1 by its plain definition (the oracle's search) on random integers."""
    rng = random.Random(7)
    for _ in range(2000):
        t_t = rng.randint(1, 500)
        t_d = rng.randint(1, t_t)
        sp = rng.randint(1, 9)
        k = rng.randint(1, 30)
        assert D.dsi_min_lookahead(t_t, t_d, sp) == O.min_lookahead(t_t, t_d, sp)
        assert D.dsi_eq1_feasible(t_t, t_d, k, sp) == int(O.eq1_feasible(t_t, t_d, k, sp))
        assert D.dsi_required_processors(t_t, t_d, k) == O.required_processors(t_t, t_d, k)
    assert D.dsi_min_lookahead(0, 1, 1) == -1


def test_shard_bounds_properties():
    rng = np.random.default_rng(0)
    for n, parts in [(0, 1), (1, 4), (10, 3), (1000, 8), (997, 7), (50, 64)]:
        c = rng.random(n) * 10
        b = D.dsi_shard_bounds(c, parts)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b.astype(np.int64)) >= 0)
        if n >= parts * 10:
            sums = [c[b[j]:b[j + 1]].sum() for j in range(parts)]
            assert max(sums) - min(sums) <= 2 * c.max() + 1e-9
    with pytest.raises(D.DsiError):
        D.dsi_shard_bounds(np.array([1.0, -1.0]), 2)


def _create(cfgs, tick=0.01, **kw):
    return D.dsi_sim_create(cfgs, tick=tick, seed=W.SEED, **kw)


def _one(**over):
    cfgs, tick = W.cfg1(trials=10)
    for k, v in over.items():
        cfgs[k] = v
    return cfgs


@pytest.mark.parametrize("over,status", [
    ({"accept_rate": 1.5}, D.DSI_E_RANGE), ({"accept_rate": -0.1}, D.DSI_E_RANGE),
    ({"accept_rate": np.nan}, D.DSI_E_RANGE), ({"lookahead": 0}, D.DSI_E_RANGE),
    ({"sp_degree": 0}, D.DSI_E_RANGE), ({"n_tokens": 0}, D.DSI_E_RANGE),
    ({"n_tokens": 40000}, D.DSI_E_RANGE), ({"n_trials": 0}, D.DSI_E_RANGE),
    ({"n_trials": (1 << 32) + 1}, D.DSI_E_RANGE), ({"t_drafter": 2.0}, D.DSI_E_RANGE),
    ({"t_target": -1.0}, D.DSI_E_RANGE), ({"t_target": np.inf}, D.DSI_E_RANGE),
    ({"t_drafter": 0.105}, D.DSI_E_TICK), ({"t_target": 0.001}, D.DSI_E_TICK),
    ({"lookahead": 10**7}, D.DSI_E_OVERFLOW), ({"n_tokens": 30000, "t_target": 1000.0}, D.DSI_E_OVERFLOW),
])
def test_create_validation_errors(over, status):
    with pytest.raises(D.DsiError) as e:
        _create(_one(**over))
    assert e.value.status == status, str(e.value)


def test_create_option_errors():
    cfgs = _one()
    bad = [dict(tick=0.0), dict(tick=-1.0), dict(flags=0x400), dict(n_devices=0), dict(n_devices=9), dict(n_devices=2),
           dict(world=2, rank=2), dict(world=0), dict(block_threads=48), dict(block_threads=256),
           dict(n_shards=2, n_devices=2), dict(flags=D.DSI_F_SHARED_STREAMS | D.DSI_F_PER_TRIAL),
           dict(flags=D.DSI_F_SHARED_STREAMS | D.DSI_F_HIST),
           dict(flags=D.DSI_F_SHARED_STREAMS | D.DSI_F_PATTERN),
           dict(flags=D.DSI_F_MEANS_ONLY | D.DSI_F_PER_TRIAL), dict(flags=D.DSI_F_MEANS_ONLY | D.DSI_F_HIST),
           dict(flags=D.DSI_F_MEANS_ONLY | D.DSI_F_PATTERN),
           dict(flags=D.DSI_F_MEANS_ONLY | D.DSI_F_SHARED_STREAMS)]
    for kw in bad:
        tick = kw.pop("tick", 0.01)
        with pytest.raises(D.DsiError) as e:
            D.dsi_sim_create(cfgs, tick=tick, seed=1, **kw)
        assert e.value.status in (D.DSI_E_RANGE, D.DSI_E_NULL), (kw, str(e.value))
    with pytest.raises(D.DsiError) as e:  # multi-GPU without an NCCL id
        D.dsi_sim_create(cfgs, tick=0.01, seed=1, world=2, rank=0)
    assert e.value.status == D.DSI_E_NULL
    with pytest.raises(D.DsiError) as e:  # per-trial records are single-device only
        D.dsi_sim_create(cfgs, tick=0.01, seed=1, world=2, rank=0, nccl_id=b"\0" * 128,
                         flags=D.DSI_F_PER_TRIAL)
    assert e.value.status == D.DSI_E_RANGE


def test_ttft_validation():
    cfgs = _one(ttft_target=1.5, ttft_drafter=2.0)  # drafter's first forward slower than target's
    with pytest.raises(D.DsiError) as e:
        _create(cfgs)
    assert e.value.status == D.DSI_E_RANGE
    with pytest.raises(D.DsiError) as e:
        _create(_one(ttft_target=1.505))
    assert e.value.status == D.DSI_E_TICK
    # TTFT configs are accepted with shared streams (they run through the per-config kernel):
    # here create gets past validation and planning and stops only for want of a GPU
    with pytest.raises(D.DsiError) as e:
        _create(_one(ttft_target=2.0), flags=D.DSI_F_SHARED_STREAMS)
    assert e.value.status == D.DSI_E_DEVICE
    with pytest.raises(D.DsiError) as e:
        _create(_one(ttft_target=2.0, n_tokens=5000))
    assert e.value.status == D.DSI_E_RANGE


def test_fresh_verifier_validation():
    with pytest.raises(D.DsiError) as e:
        _create(_one(ttft_target=2.0), flags=D.DSI_F_FRESH_VERIFIER)
    assert e.value.status == D.DSI_E_RANGE
    with pytest.raises(D.DsiError) as e:  # with shared streams too (validated, then no device here)
        _create(_one(ttft_target=2.0), flags=D.DSI_F_FRESH_VERIFIER | D.DSI_F_SHARED_STREAMS)
    assert e.value.status == D.DSI_E_RANGE


def test_shared_streams_n_limit():
    with pytest.raises(D.DsiError) as e:  # 128 run lists of N/3 + 2 u16 must fit shared memory
        _create(_one(n_tokens=2049), flags=D.DSI_F_SHARED_STREAMS)
    assert e.value.status == D.DSI_E_RANGE


def test_strict_eq1_and_pattern_limits():
    cfgs = _one(sp_degree=1)  # ceil(100 / (5*10)) = 2 > 1
    with pytest.raises(D.DsiError) as e:
        _create(cfgs, flags=D.DSI_F_STRICT_EQ1)
    assert e.value.status == D.DSI_E_STRICT_EQ1
    with pytest.raises(D.DsiError) as e:
        _create(_one(n_tokens=34), flags=D.DSI_F_PATTERN)
    assert e.value.status == D.DSI_E_RANGE
    with pytest.raises(D.DsiError):
        D.dsi_sim_create(W.cfg1()[0][:0], tick=0.01, seed=1)  # n_cfg == 0


@pytest.mark.skipif(D.lib is None, reason="no library")
def test_valid_config_without_gpu_reports_device_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(D.DsiError) as e:
        _create(W.cfg1()[0])
    assert e.value.status == D.DSI_E_DEVICE


def test_null_handles_are_rejected():
    assert D.lib.dsi_sim_run(None) == D.DSI_E_NULL
    assert D.lib.dsi_sim_reduce(None, None, 0) == D.DSI_E_NULL
    D.lib.dsi_sim_destroy(None)  # NULL-safe


def test_workloads_shapes():
    assert W.cfg1()[0].size == 1
    c2, t2 = W.cfg2()
    assert c2.size == 30 and t2 == 0.1
    c3, _ = W.cfg3(k_max=20)
    assert c3.size == 10100 * 20
    c4, _ = W.cfg4()
    assert c4.size == 140
    c5, _ = W.cfg5(D.dsi_min_lookahead)
    assert c5.size == 10100
    # every latency is a whole number of ticks (checked by the oracle's own converter)
    for c, tick in (W.cfg2(), W.cfg3(k_max=2), W.cfg5(D.dsi_min_lookahead)):
        for row in c[:: max(1, c.size // 500)]:
            O.ticks(float(row["t_target"]), tick)
            O.ticks(float(row["t_drafter"]), tick)


def test_parallel_validation_reports_the_first_bad_config():
    """Large grids are validated on the host worker pool; the error names the lowest bad index
    whatever the thread interleaving (two bad rows, the later one first in memory order)."""
    cfgs, _ = W.cfg3(k_max=20)  # 202 000 configs
    cfgs["accept_rate"][150_001] = 2.0
    cfgs["lookahead"][70_003] = 0
    for _ in range(3):
        with pytest.raises(D.DsiError) as e:
            _create(cfgs)
        assert e.value.status == D.DSI_E_RANGE
        assert "config 70003" in str(e.value), str(e.value)


def _build_c_example(tmp_path):
    import subprocess
    exe = tmp_path / "c_abi_example"
    lib_dir = os.path.join(ROOT, "paper_2405_14105_b200")
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "c_abi_example.c"), "-L" + lib_dir, "-ldsi_sim",
                        "-Wl,-rpath," + lib_dir, "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_abi_example_compiles_and_runs_without_gpu(tmp_path):
    """The README's C example builds against include/dsi_sim.h with a plain C compiler and,
    without an sm_100 device, stops at create with DSI_E_DEVICE after validating."""
    import subprocess
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present (tests/test_gpu_parity.py runs it)")
    r = subprocess.run([str(_build_c_example(tmp_path))], capture_output=True, text=True)
    assert r.returncode == 3, r.stdout + r.stderr
    assert "no device" in r.stdout


@pytest.mark.gpu
def test_c_abi_example_on_gpu(tmp_path):
    import subprocess
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([str(_build_c_example(tmp_path))], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    # expected means computed by the CPU oracle on the example's config (cfg1, tick 0.01:
    # t_t 100, t_d 10 ticks, a 0.8, k 5, SP 2, N 50, 1000 trials, seed 2405141050)
    import oracle as O
    want = O.means(O.run(O.Config(100, 10, 0.8, 5, 2, 50), 2405141050, 0, 1000, per_trial=False), 0.01)
    line = (f"mean non-SI {want['mean_nonsi']:.6f} SI {want['mean_si']:.6f} DSI {want['mean_dsi']:.6f} "
            f"over 1000 trials")
    assert line in r.stdout, (line, r.stdout)


def test_multi_drafter_options_validated_before_device_work():
    """dsi_multi_simulate rejects bad option combinations before touching a device (CPU)."""
    cfgs = W.multi_rows([(1.0, (0.1,), (0.5,))], 10, 10)
    cases = [(dict(world=2), D.DSI_E_NULL),                       # world > 1 needs an NCCL id
             (dict(world=2, rank=2, nccl_id=bytes(128)), D.DSI_E_RANGE),
             (dict(world=2, nccl_id=bytes(128), per_trial=True), D.DSI_E_RANGE),
             (dict(n_shards=2, world=2, nccl_id=bytes(128)), D.DSI_E_RANGE),
             (dict(flags=D.DSI_F_SHARED_STREAMS), D.DSI_E_RANGE)]
    for kw, status in cases:
        with pytest.raises(D.DsiError) as e:
            D.dsi_multi_simulate(cfgs, tick=0.01, seed=1, **kw)
        assert e.value.status == status, kw

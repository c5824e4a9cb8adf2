"""bench.py end to end on a small workload (the driver runs it at round end): one JSON line
with the contract's keys, every sub-block present and consistent."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line_small_workload():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "cfg2", "--steps", "2",
                        "--warmup", "3", "--cpu-seconds", "2"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks",
              "cpu_baseline", "heatmap", "shared_streams", "means_only", "multi_drafter"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["steps"] == 2 and d["warmup"] == 3
    assert 0 < d["roofline"]["frac"] <= 1.0
    assert d["heatmap"]["device_cells_equal_host_product"] is True
    assert d["shared_streams"]["bit_identical_to_value_run"] is True
    assert d["means_only"]["sums_and_means_identical_to_value_run"] is True
    assert d["multi_drafter"]["value"] > 0 and 0 < d["multi_drafter"]["roofline"]["frac"] <= 1.0
    assert 0 < d["roofline"]["fmaheavy"]["frac"] <= 1.0 and d["roofline"]["unit"] == "Ginstr/s"
    assert (d["comm"]["nranks"], d["comm"]["rank"], d["comm"]["transport"]) == (1, 0, "none")
    fv = d["heatmap"]["fresh_verifier"]
    assert fv["shared_streams_bit_identical"] is True and fv["means_only_bit_identical"] is True
    assert fv["identical_to_default_where_k_td_le_tt"] is True
    assert d["other_workloads"] is None  # (run on the cfg3 bench only)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def test_bench_two_ranks_on_one_gpu():
    """The multi-rank bench flow (torchrun, fresh ids per handle, REDUCE_TO_ROOT, max over ranks,
    every block's consistency checks) with both ranks on GPU 0: DSI_BENCH_ONE_GPU=1 puts the
    library's cross-rank sums on a gloo host all-reduce (NCCL refuses two ranks on one GPU)."""
    import socket
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, DSI_BENCH_ONE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--workload", "cfg2", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2" and d["value"] > 0
    assert (d["comm"]["nranks"], d["comm"]["rank"], d["comm"]["transport"]) == (2, 0, "host")
    # cfg2's 10 cells cannot be split in two within the 4% balance bound: the moments are exchanged
    assert d["comm"]["heatmap_exchange"] in ("cells", "moments")
    assert d["heatmap"]["fresh_verifier"]["shared_streams_bit_identical"] is True
    assert d["heatmap"]["device_cells_equal_host_product"] is True
    assert d["shared_streams"]["bit_identical_to_value_run"] is True
    assert d["means_only"]["sums_and_means_identical_to_value_run"] is True


def test_bench_gpus_flag_relaunches_itself():
    """`bench.py --gpus 2` outside torchrun re-executes itself under torch.distributed.run with
    2 processes (here both on GPU 0 through the test transport)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["DSI_BENCH_ONE_GPU"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "cfg1",
                        "--steps", "1", "--warmup", "3", "--no-multi", "--no-fresh"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 2 and d["comm"]["nranks"] == 2

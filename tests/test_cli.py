"""The command-line front end and the Table-2 protocol on top of dsi_heatmap."""
import json
import subprocess
import sys
from fractions import Fraction

import numpy as np
import pytest

import exact_math as X
from paper_2405_14105_b200 import dsi_sim as D
from paper_2405_14105_b200 import workloads as W

ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))

# Offline DSI-vs-SI speedups of the Table 2 rows in exact expectation under DESIGN.md's reading
# (N = 100, SP = 8, lookahead in {1, 5, 10}); BASELINE.md section 2 lists the same values.
# Context, not paper numbers: the paper's online speedups are 1.29-1.92.
TABLE2_EXACT = [1.40, 1.44, 1.25, 1.22, 1.26, 1.25, 1.15, 1.16, 1.18, 1.18]


def run_cli(*args):
    r = subprocess.run([sys.executable, "-m", "paper_2405_14105_b200", *args], capture_output=True,
                       text=True, cwd=ROOT)
    return r.returncode, r.stdout, r.stderr


def test_plan_matches_paper_examples():
    rc, out, _ = run_cli("plan", "--t-target", "1.0", "--t-drafter", "0.05", "--sp", "4")
    assert rc == 0
    d = json.loads(out)
    assert d["min_lookahead"] == 5 and d["processors"] == 5
    rc, out, _ = run_cli("plan", "--t-target", "1.0", "--t-drafter", "0.05", "--sp", "3")
    assert json.loads(out)["min_lookahead"] == 7


def test_plan_validates_like_create():
    """plan converts latencies with the library's R15 rule (dsi_ticks) and checks Assumption 2:
    a non-whole number of ticks, a nonpositive latency or t_drafter > t_target exit 2."""
    rc, _, err = run_cli("plan", "--t-target", "1.0", "--t-drafter", "0.004", "--sp", "4")
    assert rc == 2 and "DSI_E_TICK" in err
    rc, _, err = run_cli("plan", "--t-target", "-1.0", "--t-drafter", "0.05", "--sp", "4")
    assert rc == 2 and "DSI_E_RANGE" in err
    rc, _, err = run_cli("plan", "--t-target", "0.5", "--t-drafter", "1.0", "--sp", "4")
    assert rc == 2 and "Assumption 2" in err
    rc, _, err = run_cli("plan", "--t-target", "1.0", "--t-drafter", "0.05", "--sp", "0")
    assert rc == 2
    rc, out, _ = run_cli("plan", "--t-target", "1.0", "--t-drafter", "0.1", "--sp", "2")
    d = json.loads(out)
    assert rc == 0 and d["max_useful_sp"] == 10 and d["min_lookahead"] == 5 and d["processors"] == 3


def test_ticks_rule():
    assert D.dsi_ticks(0.3, 0.1) == 3 and D.dsi_ticks(20.6, 0.1) == 206
    for x, tick, st in ((0.004, 0.01, D.DSI_E_TICK), (0.0, 0.01, D.DSI_E_RANGE), (1.0, -0.01, D.DSI_E_RANGE),
                        (float("nan"), 0.01, D.DSI_E_RANGE)):
        with pytest.raises(D.DsiError) as e:
            D.dsi_ticks(x, tick)
        assert e.value.status == st


def test_invalid_arguments_exit_2():
    rc, _, err = run_cli("simulate", "--t-target", "1.0", "--t-drafter", "2.0", "--accept", "0.5",
                         "--lookahead", "1", "--sp", "2", "--n-tokens", "10")
    assert rc == 2 and "DSI_E_RANGE" in err


def exact_results(cfgs, tick):
    res = np.zeros(cfgs.size, D.RESULT_DTYPE)
    for i, row in enumerate(cfgs):
        t_t, t_d = round(row["t_target"] / tick), round(row["t_drafter"] / tick)
        k, sp, N = int(row["lookahead"]), int(row["sp_degree"]), int(row["n_tokens"])
        p = Fraction(int(float(row["accept_rate"]) * 2 ** 32), 2 ** 32)
        e = X.expectations(N, k, t_d, t_t, sp, p)
        res[i]["mean_si"] = float(e["si"]) * tick
        res[i]["mean_dsi"] = float(e["dsi"]) * tick
        res[i]["mean_nonsi"] = N * t_t * tick
        res[i]["eq1_feasible"] = int(-(-t_t // (k * t_d)) <= sp)
    return res


def test_table2_protocol_exact():
    """SI best over {1,5,10}, DSI best over the Eq.-1-feasible subset, speedup SI/DSI."""
    cfgs, tick = W.cfg2()
    cells = D.dsi_heatmap(cfgs, exact_results(cfgs, tick))
    assert cells.size == 10
    assert [round(float(c), 2) for c in cells["r_si_dsi"]] == TABLE2_EXACT
    # the Vicuna rows cannot use k = 1 on 8 servers (Eq. 1: ceil(377/25) = 16 > 8)
    assert list(cells["dsi_lookahead"][6:]) == [5, 5, 5, 5]


@pytest.mark.gpu
def test_table2_monte_carlo_on_gpu():
    from paper_2405_14105_b200.cli import table2
    rows = table2(trials=100_000, sp=8, n_tokens=100)
    got = [r["speedup_dsi_vs_si"] for r in rows]
    assert np.allclose(got, TABLE2_EXACT, atol=0.012), got


@pytest.mark.gpu
def test_heatmap_cli_writes_csv(tmp_path):
    path = tmp_path / "heat.csv"
    rc, out, err = run_cli("heatmap", "--trials", "300", "--k-max", "12", "--csv", str(path), "--shared")
    assert rc == 0, err
    d = json.loads(out)
    assert d["cells"] == 10100
    lines = path.read_text().splitlines()
    assert len(lines) == 2 + 10100


@pytest.mark.gpu
def test_simulate_fresh_verifier_cli():
    """k t_d > t_t: the default model can lose to non-SI; the fresh-verifier variant cannot
    (Thm 1 per trial, R24)."""
    args = ["simulate", "--t-target", "1.0", "--t-drafter", "1.0", "--accept", "0.48", "--lookahead", "20",
            "--sp", "7", "--n-tokens", "100", "--trials", "20000"]
    rc, out, err = run_cli(*args)
    assert rc == 0, err
    base = json.loads(out)
    rc, out, err = run_cli(*args, "--fresh")
    assert rc == 0, err
    fresh = json.loads(out)
    assert base["mean_dsi"] > base["mean_nonsi"]          # R5: E[non-SI]/E[DSI] = 0.18
    assert fresh["n_dsi_gt_nonsi"] == 0 and fresh["mean_dsi"] <= fresh["mean_nonsi"]
    assert fresh["sum_si_ticks"] == base["sum_si_ticks"]   # SI is unchanged


@pytest.mark.gpu
def test_fig5_static_lookahead_monte_carlo(tmp_path):
    """Fig. 5 by Monte Carlo through the CLI: lookahead 5, fresh-verifier DSI.
    DSI is never slower than non-SI (per trial, so exactly in the means) and not slower than
    SI beyond Monte Carlo noise; SI is slower than non-SI on about 7266 cells (exact count)."""
    path = tmp_path / "fig5.csv"
    rc, out, err = run_cli("heatmap", "--trials", "4000", "--k", "5", "--fresh", "--csv", str(path))
    assert rc == 0, err
    rows = np.genfromtxt(path, delimiter=",", skip_header=2)
    r_nonsi_si, r_si_dsi, r_nonsi_dsi = rows[:, 7], rows[:, 8], rows[:, 9]
    ok = ~np.isnan(r_nonsi_dsi)  # t_d in {0.01, 0.02}: Eq. 1 fails at k = 5, SP = 7 (no DSI value)
    assert ok.sum() == 10100 - 2 * 101
    assert np.all(r_nonsi_dsi[ok] >= 1.0)
    assert np.all(r_si_dsi[ok] >= 0.99)
    assert abs(int(np.sum(r_nonsi_si < 1.0)) - 7266) < 150


def test_multi_cli_rejects_unordered_drafters():
    rc, out, err = run_cli("multi", "--t-target", "1.0", "--drafter", "0.2:0.5", "--drafter", "0.1:0.5",
                           "--n-tokens", "10", "--trials", "10")
    assert rc == 2 and "ordered by latency" in err


@pytest.mark.gpu
def test_multi_cli_expectation():
    """Two drafters, lookahead 1: E[L] = t_m + (N-1) sum_j t_j pi_j, pi = (a_1,
    (1-a_1) a_2, (1-a_1)(1-a_2)); 1e5 trials within 6 sigma (sigma from the per-position law)."""
    rc, out, err = run_cli("multi", "--t-target", "1.0", "--drafter", "0.02:0.5", "--drafter", "0.1:0.8",
                           "--n-tokens", "100", "--trials", "100000")
    assert rc == 0, err
    r = json.loads(out)
    pi = [0.5, 0.5 * 0.8, 0.5 * 0.2]
    lat = [0.02, 0.1, 1.0]
    e1 = sum(p * t for p, t in zip(pi, lat))
    e2 = sum(p * t * t for p, t in zip(pi, lat))
    mean, sd = 1.0 + 99 * e1, (99 * (e2 - e1 * e1)) ** 0.5
    assert abs(r["mean_dsi"] - mean) <= 6 * sd / 100000 ** 0.5
    assert r["n_dsi_gt_nonsi"] == 0 and r["models"] == 3


@pytest.mark.gpu
def test_heatmap_cli_means_only_matches_shared(tmp_path):
    """--means (segment histograms) writes the same CSV as --shared (per-trial evaluation)."""
    a, b = tmp_path / "means.csv", tmp_path / "shared.csv"
    for path, flag in ((a, "--means"), (b, "--shared")):
        rc, out, err = run_cli("heatmap", "--trials", "400", "--k-max", "20", "--csv", str(path), flag)
        assert rc == 0, err
    assert a.read_text() == b.read_text()


@pytest.mark.gpu
def test_heatmap_cli_under_torchrun_matches_one_process(tmp_path):
    """The CLI heatmap sharded over 2 ranks (torchrun; both on GPU 0 through the host all-reduce
    hook, DSI_BENCH_ONE_GPU=1) writes the same CSV as one process."""
    import os
    import socket
    one, two = tmp_path / "one.csv", tmp_path / "two.csv"
    rc, out, err = run_cli("heatmap", "--trials", "500", "--k-max", "20", "--means", "--csv", str(one))
    assert rc == 0, err
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "-m", "paper_2405_14105_b200",
                        "heatmap", "--trials", "500", "--k-max", "20", "--means", "--csv", str(two)],
                       capture_output=True, text=True, cwd=ROOT, env=dict(os.environ, DSI_BENCH_ONE_GPU="1"),
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert one.read_text() == two.read_text()
    assert json.loads(r.stdout)["cells"] == 10100

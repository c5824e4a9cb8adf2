"""The heatmap product (Fig. 3, App. F.3) on CPU.

dsi_heatmap is a host-only function of the library, so it is tested here with result
arrays built from the EXACT expectations (tests/exact_math.py) of the paper's grid: the
argmin over lookaheads, the Eq.-1 filter for DSI and the four ratio panels, plus the
paper-level claims the grid must show (P14, P16 of SURVEY 8(c).5).
"""
from fractions import Fraction

import numpy as np
import pytest

import exact_math as X
from paper_2405_14105_b200 import dsi_sim as D
from paper_2405_14105_b200 import workloads as W


def exact_results(cfgs, tick, N=100, sp=7, t_t=100):
    """dsi_result rows whose means are the exact expectations at the realised p = thr / 2^32."""
    t_d_axis = np.array(sorted(set(np.rint(cfgs["t_drafter"] / tick).astype(int))))
    a_axis = np.array(sorted(set(cfgs["accept_rate"].tolist())))
    k_axis = np.array(sorted(set(cfgs["lookahead"].tolist())))
    thr = np.floor(a_axis * 4294967296.0)
    e_si, e_dsi = X.expectations_grid_f64(N, t_t, t_d_axis, k_axis, sp, thr / 4294967296.0)
    res = np.zeros(cfgs.size, D.RESULT_DTYPE)
    ia = np.searchsorted(a_axis, cfgs["accept_rate"])
    idd = np.searchsorted(t_d_axis, np.rint(cfgs["t_drafter"] / tick).astype(int))
    ik = np.searchsorted(k_axis, cfgs["lookahead"])
    res["mean_si"] = e_si[ia, idd, ik] * tick
    res["mean_dsi"] = e_dsi[ia, idd, ik] * tick
    res["mean_nonsi"] = N * t_t * tick
    td = t_d_axis[idd]
    res["eq1_feasible"] = (-(-t_t // (cfgs["lookahead"] * td)) <= sp).astype(np.int32)
    return res


def test_grid_expectations_match_fractions():
    """The vectorised float64 expectation equals the exact rational one."""
    e_si, e_dsi = X.expectations_grid_f64(30, 100, [7, 30], [1, 2, 5], 3, [0.0, 0.6, 1.0])
    for ip, p in enumerate([0, Fraction(3, 5), 1]):
        for idd, td in enumerate([7, 30]):
            for ik, k in enumerate([1, 2, 5]):
                e = X.expectations(30, k, td, 100, 3, p)
                assert abs(e_dsi[ip, idd, ik] - float(e["dsi"])) < 1e-9 * float(e["dsi"])
                assert abs(e_si[ip, idd, ik] - float(e["si"])) < 1e-9 * float(e["si"])


def test_heatmap_argmin_and_ratios_small():
    cfgs, tick = W.cfg3(k_max=12, cells=slice(0, 10100, 97))
    res = exact_results(cfgs, tick)
    cells = D.dsi_heatmap(cfgs, res)
    assert cells.size == cfgs.size // 12
    for c in cells:
        sl = slice(int(c["first_cfg"]), int(c["first_cfg"] + c["n_cfg"]))
        si = res["mean_si"][sl]
        assert c["si"] == si.min() and c["si_lookahead"] == cfgs["lookahead"][sl][np.argmin(si)]
        feas = res["eq1_feasible"][sl] == 1
        if feas.any():
            dsi = np.where(feas, res["mean_dsi"][sl], np.inf)
            assert c["dsi"] == dsi.min() and c["dsi_lookahead"] == cfgs["lookahead"][sl][np.argmin(dsi)]
            assert c["r_min_dsi"] == min(c["si"], c["nonsi"]) / c["dsi"]
        else:
            assert c["dsi_lookahead"] == -1 and np.isnan(c["dsi"])
        assert c["r_nonsi_si"] == c["nonsi"] / c["si"]


def test_heatmap_ties_go_to_smallest_lookahead(tmp_path):
    cfgs, _ = W.cfg3(k_max=4, cells=slice(0, 2))
    res = np.zeros(cfgs.size, D.RESULT_DTYPE)
    res["mean_si"] = 5.0
    res["mean_dsi"] = 3.0
    res["mean_nonsi"] = 10.0
    res["eq1_feasible"] = [0, 1, 1, 1, 0, 0, 0, 0]
    cells = D.dsi_heatmap(cfgs, res)
    assert list(cells["si_lookahead"]) == [1, 1]
    assert list(cells["dsi_lookahead"]) == [2, -1]
    p = tmp_path / "h.csv"
    D.dsi_heatmap_csv(cells, str(p))
    lines = p.read_text().splitlines()
    assert lines[0].startswith("# dsi_heatmap v1")
    assert lines[1].split(",")[:3] == ["drafter_latency", "acceptance_rate", "nonsi"]
    assert lines[2] == "0.010000,0.000000,10.000000,5.000000,3.000000,1,2,2.000000,1.666667,3.333333,1.666667"
    assert len(lines) == 4


@pytest.fixture(scope="module")
def full_grid():
    cfgs, tick = W.cfg3()
    return cfgs, tick, D.dsi_heatmap(cfgs, exact_results(cfgs, tick))


def test_fig3a_si_faster_than_nonsi_iff_acceptance_exceeds_drafter_latency(full_grid):
    """P14: in exact expectation SI beats non-SI exactly where a > t_d/t_t,
    on all 10 100 cells (N = 100, SI lookahead 1..200)."""
    cfgs, tick, cells = full_grid
    assert cells.size == 10100
    faster = cells["r_nonsi_si"] > 1.0
    assert np.array_equal(faster, cells["accept_rate"] > cells["t_drafter"] / cells["t_target"])


def test_fig3bcd_dsi_never_slower(full_grid):
    """P16: non-SI/DSI >= 1 everywhere; SI/DSI >= 1 except where Eq. 1 forces a large
    DSI lookahead at t_d = 0.01; max min(SI, non-SI)/DSI ~ 1.53 (paper: 'up to 1.6x')."""
    _, _, cells = full_grid
    assert np.all(cells["dsi_lookahead"] >= 1)
    assert np.all(cells["r_nonsi_dsi"] >= 1.0 - 1e-12)
    bad = cells[cells["r_si_dsi"] < 1.0]
    assert bad.size == 46 and np.all(np.isclose(bad["t_drafter"], 0.01))
    assert 0.99 < bad["r_si_dsi"].min() < 1.0
    i = np.argmax(cells["r_min_dsi"])
    assert abs(cells["r_min_dsi"][i] - 1.528) < 0.001
    assert np.isclose(cells["t_drafter"][i], 0.15) and np.isclose(cells["accept_rate"][i], 0.91)
    assert cells["si_lookahead"][i] == 8 and cells["dsi_lookahead"][i] == 1


def test_fresh_grid_matches_scalar_closed_form():
    e_si, e_dsi = X.expectations_grid_f64(40, 100, [7, 30, 100], [1, 5, 20], 3, [0.0, 0.6, 1.0], fresh=True)
    for ip, p in enumerate([0, Fraction(3, 5), 1]):
        for idd, td in enumerate([7, 30, 100]):
            for ik, k in enumerate([1, 5, 20]):
                e = X.expectations_fresh(40, k, td, 100, 3, p)
                assert abs(e_dsi[ip, idd, ik] - float(e["dsi"])) < 1e-9 * float(e["dsi"])


def test_fig5_static_lookahead_needs_the_fresh_verifier():
    """App. F.5 / Fig. 5: with SI and DSI at lookahead 5 (N = 100, SP = 7),
    "SI is slower than non-SI when the drafter is either slow or inaccurate enough" and
    "DSI is never slower than either SI or non-SI".  Exact expectations on all 10 100 cells:
    the fresh-verifier variant (R24) meets both claims everywhere; the default
    model (R5) is slower than non-SI on 5497 cells, all with k t_d > t_t."""
    t_d = np.arange(1, 101)
    ps = np.arange(0, 101) / 100
    non = 100 * 100.0
    for fresh in (False, True):
        e_si, e_dsi = X.expectations_grid_f64(100, 100, t_d, [5], 7, ps, fresh=fresh)
        e_si, e_dsi = e_si[:, :, 0], e_dsi[:, :, 0]
        assert int(np.sum(e_si > non * (1 + 1e-12))) == 7266            # Fig. 5(a) pink cells
        assert np.all(e_dsi <= e_si * (1 + 1e-12))                       # Fig. 5(b)
        slower = e_dsi > non * (1 + 1e-12)                               # Fig. 5(c)
        if fresh:
            assert not slower.any()
        else:
            assert int(slower.sum()) == 5497
            assert np.all(5 * t_d[np.nonzero(slower)[1]] > 100)

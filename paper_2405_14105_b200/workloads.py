"""Seeded synthetic inputs: the configuration grids of BASELINE.json ``configs``.

Shared by the product tests, bench.py and the oracle-side tests.  It holds none
of the method's arithmetic: it only lists grid points in user units (the
paper's quantities) as numpy arrays with the C layout of ``dsi_config``.  Where
a grid needs a lookahead chosen by Eq. 1 (config 5) the caller passes the
planner in (``k_of_cell``).

Recipe:
  * seed 2405141050 (0x8F5B8A3A, from the arXiv id); stream_id 0 everywhere
    (common random numbers across configs);
  * cfg1  single point   t_t 1.0, t_d 0.1, a 0.8, k 5, SP 2, N 50, T 1e3, tick 0.01;
  * cfg2  Table 2 pairs in ms, tick 0.1 ms, SP 8, N 100, k in {1,5,10}, T 1e5;
  * cfg3  heatmap        t_t 1.0, t_d in {0.01..1.00}, a in {0.00..1.00},
                         k in 1..200 ("fast" variant 1..20), SP 7, N 100, T 1e4;
  * cfg4  k x SP sweep   t_t 1.0, t_d 0.1, a 0.8, k 1..20, SP 2..8, N 500, T 1e5;
  * cfg5  large MC       cfg3's 10 100 cells at SP 7 with k = k_of_cell, N 1000, T 1e5.
Acceptance is i.i.d. Bernoulli(a) per draft, drawn inside the simulator
from the Philox stream keyed by the seed.
"""
from __future__ import annotations

import numpy as np

SEED = 2405141050

CONFIG_DTYPE = np.dtype([("t_target", "<f8"), ("t_drafter", "<f8"), ("accept_rate", "<f8"),
                         ("lookahead", "<i4"), ("sp_degree", "<i4"), ("n_tokens", "<i4"),
                         ("stream_id", "<u4"), ("n_trials", "<u8"), ("ttft_target", "<f8"),
                         ("ttft_drafter", "<f8")])

# Table 2: target latency ms, drafter latency ms, acceptance rate.
TABLE2_ROWS = [
    ("Starcoder-15B/168M HumanEval", 20.6, 6.8, 0.93),
    ("Starcoder-15B/168M MBPP", 21.0, 6.8, 0.90),
    ("Phi3-14B/4B Alpaca", 49.6, 33.4, 0.87),
    ("Phi3-14B/4B HumanEval", 52.1, 34.0, 0.95),
    ("Phi3-14B/4B CNN-DM", 52.4, 34.6, 0.93),
    ("Phi3-14B/4B MBPP", 52.2, 34.3, 0.94),
    ("Vicuna-13B/68M CNN-DM", 37.7, 2.5, 0.63),
    ("Vicuna-13B/68M Alpaca", 33.3, 2.5, 0.58),
    ("Vicuna-7B/68M CNN-DM", 29.4, 2.5, 0.67),
    ("Vicuna-7B/68M Alpaca", 26.0, 2.5, 0.59),
]


# Table 3: TTFT/TPOT ratios of (target, drafter) per Table-2 row; the Phi-3
# Alpaca row has no Table-3 entry and keeps TTFT = TPOT (ratio 1).
TABLE3_TTFT_RATIOS = [(1.35, 1.19), (1.54, 1.20), (1.0, 1.0), (1.29, 1.23), (4.77, 3.88),
                      (1.43, 1.27), (5.36, 1.04), (1.15, 1.05), (4.53, 1.06), (1.19, 1.06)]


def _grid(rows) -> np.ndarray:
    """Rows (t_target, t_drafter, a, k, SP, N, stream_id, T[, ttft_target, ttft_drafter])."""
    out = np.zeros(len(rows), CONFIG_DTYPE)
    for i, r in enumerate(rows):
        out[i] = tuple(r) + (0.0, 0.0)[: 10 - len(r)]
    return out


rows = _grid  # public name for tests and tools


def cfg1(trials: int = 1000):
    """BASELINE configs[0]: the single point the oracle finishes in seconds."""
    return _grid([(1.0, 0.1, 0.8, 5, 2, 50, 0, trials)]), 0.01


def cfg2(trials: int = 100_000, sp: int = 8, n_tokens: int = 100, ks=(1, 5, 10)):
    """BASELINE configs[1]: Table-2 (target, drafter, task) pairs; tick 0.1 ms."""
    rows = [(tt, td, a, k, sp, n_tokens, 0, trials) for _, tt, td, a in TABLE2_ROWS for k in ks]
    return _grid(rows), 0.1


def cfg2_ttft(trials: int = 10_000, sp: int = 7, n_tokens: int = 50, ks=(1, 5, 10)):
    """The Table-2 protocol with prefill (50 tokens, "including prefilling", up to 8
    GPUs -> SP 7, k in {1,5,10}): first forwards cost TTFT = Table-3 ratio x TPOT (SURVEY
    8(f) N2).  tick 0.001 ms makes every ratio x TPOT a whole number of ticks."""
    rows = []
    for (_, tt, td, a), (rt, rd) in zip(TABLE2_ROWS, TABLE3_TTFT_RATIOS):
        for k in ks:
            rows.append((tt, td, a, k, sp, n_tokens, 0, trials, rt * tt, rd * td))
    return _grid(rows), 0.001


def heatmap_axes():
    """Drafter latency {0.01..1.00} x acceptance {0.00..1.00}."""
    t_d = np.array([i / 100 for i in range(1, 101)])
    acc = np.array([i / 100 for i in range(0, 101)])
    return t_d, acc


def cfg3(trials: int = 10_000, k_max: int = 200, sp: int = 7, n_tokens: int = 100,
         cells: slice | None = None, k_min: int = 1):
    """BASELINE configs[2]: the heatmap, every (t_d, a, k) point; order t_d-major, then a, then k.
    k_min = k_max = 5 gives the static-lookahead panels of Fig. 5."""
    t_d, acc = heatmap_axes()
    n_cells = t_d.size * acc.size
    ks = np.arange(k_min, k_max + 1, dtype=np.int32)
    cell_idx = np.arange(n_cells)
    if cells is not None:
        cell_idx = cell_idx[cells]
    out = np.zeros(cell_idx.size * ks.size, CONFIG_DTYPE)
    ci = np.repeat(cell_idx, ks.size)
    out["t_target"] = 1.0
    out["t_drafter"] = t_d[ci // acc.size]
    out["accept_rate"] = acc[ci % acc.size]
    out["lookahead"] = np.tile(ks, cell_idx.size)
    out["sp_degree"] = sp
    out["n_tokens"] = n_tokens
    out["stream_id"] = 0
    out["n_trials"] = trials
    return out, 0.01


def cfg4(trials: int = 100_000, n_tokens: int = 500):
    """BASELINE configs[3]: k = 1..20 x SP = 2..8 at config 1's (t_t, t_d, a)."""
    rows = [(1.0, 0.1, 0.8, k, sp, n_tokens, 0, trials) for k in range(1, 21) for sp in range(2, 9)]
    return _grid(rows), 0.01


def cfg5(k_of_cell, trials: int = 100_000, n_tokens: int = 1000, sp: int = 7):
    """BASELINE configs[4]: the heatmap cells at SP 7, k chosen per cell by ``k_of_cell``.

    k_of_cell(t_target_ticks, t_drafter_ticks, sp) -> k, e.g. the Eq. 1 planner."""
    t_d, acc = heatmap_axes()
    rows = []
    for td in t_d:
        k = int(k_of_cell(100, int(round(td * 100)), sp))
        for a in acc:
            rows.append((1.0, td, a, k, sp, n_tokens, 0, trials))
    return _grid(rows), 0.01


def subsample(configs: np.ndarray, n: int) -> np.ndarray:
    """n evenly spaced configs (the oracle's sampled parity / timing set)."""
    if configs.size <= n:
        return configs.copy()
    idx = np.unique(np.linspace(0, configs.size - 1, n).round().astype(np.int64))
    return configs[idx].copy()


def fuzz(n: int, seed: int = 5, n_max: int = 60, trials: int = 64):
    """Random configs covering the edge cases: SP 1..8, k 1..12 (and k > N), t_d in [1, t_t],
    N in {1, 2, 3, ...}, a in {0, 1, random}; latencies in integer ticks (tick 1)."""
    rng = np.random.default_rng(seed)
    out = np.zeros(n, CONFIG_DTYPE)
    for i in range(n):
        t_t = int(rng.integers(1, 121))
        t_d = int(rng.integers(1, t_t + 1))
        N = int(rng.choice([1, 2, 3, int(rng.integers(1, n_max + 1)), int(rng.integers(1, n_max + 1))]))
        a = float(rng.choice([0.0, 1.0, rng.random(), rng.random()]))
        k = int(rng.integers(1, 13))
        if i % 17 == 0:
            k = N + int(rng.integers(1, 5))  # lookahead beyond N
        out[i] = (float(t_t), float(t_d), a, k, int(rng.integers(1, 9)), N,
                  int(rng.integers(0, 4)), trials, 0.0, 0.0)
    return out, 1.0


# ---- multi-drafter DSI: Algorithm 1 with m models, lookahead 1 ----------
MAX_DRAFTERS = 7
MULTI_CONFIG_DTYPE = np.dtype([("t_target", "<f8"), ("t_drafter", "<f8", (MAX_DRAFTERS,)),
                               ("accept_rate", "<f8", (MAX_DRAFTERS,)), ("n_drafters", "<i4"),
                               ("n_tokens", "<i4"), ("stream_id", "<u4"), ("reserved", "<u4"),
                               ("n_trials", "<u8")])


def multi_rows(rows, trials: int, n_tokens: int, stream_id: int = 0) -> np.ndarray:
    """rows: (t_target, (t_1, ..., t_{m-1}), (a_1, ..., a_{m-1})) in user units."""
    out = np.zeros(len(rows), MULTI_CONFIG_DTYPE)
    for i, (tt, tds, rates) in enumerate(rows):
        out[i]["t_target"] = tt
        out[i]["t_drafter"][:len(tds)] = tds
        out[i]["accept_rate"][:len(rates)] = rates
        out[i]["n_drafters"] = len(tds)
    out["n_tokens"] = n_tokens
    out["n_trials"] = trials
    out["stream_id"] = stream_id
    return out


def multi_heatmap(trials: int = 10_000, n_tokens: int = 100, t_fast: float = 0.01, a_fast: float = 0.5):
    """cfg3's (drafter latency, acceptance) grid as drafter f_2 of m = 3 models, with a
    fast drafter f_1 (t_fast <= every t_d, acceptance a_fast) in front: 10 100 configs, tick 0.01."""
    t_ds, rates = heatmap_axes()
    rows = [(1.0, (t_fast, float(td)), (a_fast, float(a))) for td in t_ds for a in rates]
    return multi_rows(rows, trials, n_tokens), 0.01


def multi_fuzz(n: int, seed: int = 9, n_max: int = 60, trials: int = 64):
    """Random m in 2..8, latencies on a 1-tick grid (tick 1), ordered drafters, a in [0, 1]
    with exact 0 and 1 mixed in, ragged N and trial counts."""
    rng = np.random.default_rng(seed)
    rows, Ns, Ts = [], [], []
    for _ in range(n):
        m = int(rng.integers(2, 9))
        tt = int(rng.integers(1, 120))
        tds = sorted(int(x) for x in rng.integers(1, tt + 1, size=m - 1))
        rates = [float(x) for x in rng.random(m - 1)]
        for j in range(m - 1):
            u = rng.random()
            if u < 0.1:
                rates[j] = 0.0
            elif u < 0.2:
                rates[j] = 1.0
        rows.append((float(tt), tuple(float(x) for x in tds), tuple(rates)))
        Ns.append(int(rng.integers(1, n_max + 1)))
        Ts.append(int(rng.integers(1, trials + 1)))
    out = multi_rows(rows, 1, 1)
    out["n_tokens"] = Ns
    out["n_trials"] = Ts
    out["stream_id"] = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    return out, 1.0

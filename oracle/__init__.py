"""CPU oracle of the DSI Monte Carlo latency simulator (arXiv 2405.14105).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product (``include/dsi_sim.h`` + ``paper_2405_14105_b200``) never
imports it and shares no code with it.

The arithmetic lives in ``dsi_oracle.c`` (plain C, single-threaded): the SI
pseudocode loop of App. F.4 and an event simulation of
Algorithm 1 with the App. D lookahead.  This module only
marshals arguments through ctypes and converts user units to integer ticks.

Pins (tests/test_oracle_pins.py): Philox known-answer vectors, Table 1,
Proposition 1, Theorem 1, the non-SI example,
the SI closed form E[n+1] = (1-a^{k+1})/(1-a), exhaustive
enumeration of acceptance patterns against exact rational expectations, and
hand-derived worked examples; the halves indicator layout (R26) by
tests/test_oracle_halves.py (equal to the plain 32-bit comparison of the concatenated
halves, forced ties both ways, the Bernoulli law where every acceptance or rejection is a
tie).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dsi_oracle.c")
_SRC_MULTI = os.path.join(_HERE, "dsi_oracle_multi.c")
_HDR = os.path.join(_HERE, "dsi_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no intrinsics)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB) for s in (_SRC, _SRC_MULTI, _HDR))
    if force or stale:
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, _SRC_MULTI])
    return _LIB


class _Config(ctypes.Structure):
    _fields_ = [("t_target", ctypes.c_int64), ("t_drafter", ctypes.c_int64),
                ("accept_rate", ctypes.c_double), ("lookahead", ctypes.c_int32),
                ("sp_degree", ctypes.c_int32), ("n_tokens", ctypes.c_int32),
                ("stream_id", ctypes.c_uint32), ("t_target_first", ctypes.c_int64),
                ("t_drafter_first", ctypes.c_int64), ("fresh_verifier", ctypes.c_int32),
                ("rng_halves", ctypes.c_int32)]


class _TrialOut(ctypes.Structure):
    _fields_ = [("acc", ctypes.c_int32), ("m", ctypes.c_int32), ("iters", ctypes.c_int32),
                ("nonsi", ctypes.c_int64), ("si", ctypes.c_int64), ("dsi", ctypes.c_int64),
                ("dsi_segments", ctypes.c_int32), ("dsi_peak_busy", ctypes.c_int32),
                ("dsi_max_queue", ctypes.c_int32), ("dsi_forwards", ctypes.c_int32)]


class _Sums(ctypes.Structure):
    _fields_ = [("trials", ctypes.c_uint64), ("sum_acc", ctypes.c_int64),
                ("sum_m", ctypes.c_int64), ("sum_iters", ctypes.c_int64),
                ("sum_si", ctypes.c_int64), ("sum_dsi", ctypes.c_int64),
                ("sumsq_si", ctypes.c_uint64), ("sumsq_dsi", ctypes.c_uint64),
                ("n_dsi_gt_nonsi", ctypes.c_int64), ("n_dsi_gt_si", ctypes.c_int64)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        lib.oracle_philox4x32_10.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
        lib.oracle_philox4x32_10.restype = None
        lib.oracle_threshold.argtypes = [ctypes.c_double]
        lib.oracle_threshold.restype = ctypes.c_uint64
        lib.oracle_trial.argtypes = [P(_Config), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                     P(_TrialOut), ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_trial.restype = ctypes.c_int
        lib.oracle_trace_trial.argtypes = [P(_Config), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                           P(_TrialOut), ctypes.c_char_p, ctypes.c_size_t, P(ctypes.c_size_t)]
        lib.oracle_trace_trial.restype = ctypes.c_int
        lib.oracle_run.argtypes = [P(_Config), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_int, P(_Sums)] + [ctypes.c_void_p] * 7
        lib.oracle_run.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclass(frozen=True)
class Config:
    """One grid point in integer ticks (the paper's quantities, Table 2 cols P:249-256)."""
    t_target: int
    t_drafter: int
    accept_rate: float
    lookahead: int
    sp_degree: int
    n_tokens: int
    stream_id: int = 0
    t_target_first: int = 0   # TTFT variant: 0 = same as t_target
    t_drafter_first: int = 0  # TTFT variant: 0 = same as t_drafter
    fresh_verifier: bool = False  # N4 variant (R24)
    rng_halves: bool = False  # the halves layout of the indicator stream (R26)

    def _c(self) -> _Config:
        return _Config(int(self.t_target), int(self.t_drafter), float(self.accept_rate),
                       int(self.lookahead), int(self.sp_degree), int(self.n_tokens),
                       int(self.stream_id), int(self.t_target_first), int(self.t_drafter_first),
                       int(bool(self.fresh_verifier)), int(bool(self.rng_halves)))


def ticks(x: float, tick: float) -> int:
    """User latency -> integer ticks: round(x/tick), must be within 1e-9 relative."""
    r = x / tick
    t = int(round(r))
    if t < 1 or abs(r - t) > 1e-9 * abs(r):
        raise ValueError(f"latency {x} is not an integer number of ticks of {tick}")
    return t


def philox4x32_10(ctr, key):
    lib = _load()
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib.oracle_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def threshold(a: float) -> int:
    return int(_load().oracle_threshold(float(a)))


def trial(cfg: Config, seed: int, index: int, pattern: bool = False, hist: bool = False) -> dict:
    """One trial: acc, m, iters, nonsi, si, dsi (+ event-sim debug counters)."""
    lib = _load()
    out = _TrialOut()
    si_hist = np.zeros(cfg.lookahead + 1, np.int64) if hist else None
    seg_hist = np.zeros(64, np.int64) if hist else None
    rc = lib.oracle_trial(ctypes.byref(cfg._c()), seed, index, int(pattern), ctypes.byref(out),
                          si_hist.ctypes.data if hist else None,
                          seg_hist.ctypes.data if hist else None)
    if rc:
        raise ValueError(f"oracle_trial failed for {cfg}")
    d = {f: getattr(out, f) for f, _ in _TrialOut._fields_}
    if hist:
        d["si_hist"], d["seg_hist"] = si_hist, seg_hist
    return d


# The documented total order of trace events (SPEC S:178 asks for one): time, then segment (a
# rejection at t ends segment s before segment s+1 starts at t), then kind in this order --
# releases before claims at equal times (R8) -- then position and thread
TRACE_KINDS = ("SegmentStart", "DraftDone", "VerifyDone", "ServerFreed", "Accept", "Reject", "TokenEmitted",
               "VerifyQueued", "VerifyDispatch", "FreshDispatch")


def trace(cfg: Config, seed: int, index: int, pattern: bool = False, cap: int = 1 << 22) -> tuple:
    """One trial's DSI event trace (Fig. 1-style timeline; debug output):
    (trial record as trial(), events in TRACE_KINDS' total order).  Times in
    ticks; thread -1 = no verification thread (drafts, fresh forwards, segment starts)."""
    import json

    lib = _load()
    out = _TrialOut()
    buf = ctypes.create_string_buffer(cap)
    n = ctypes.c_size_t()
    rc = lib.oracle_trace_trial(ctypes.byref(cfg._c()), seed, index, int(pattern), ctypes.byref(out), buf, cap,
                                ctypes.byref(n))
    if rc:
        raise ValueError(f"oracle_trace_trial failed ({rc}) for {cfg}")
    events = [json.loads(ln) for ln in buf.raw[:n.value].decode().splitlines()]
    order = {k: i for i, k in enumerate(TRACE_KINDS)}
    events.sort(key=lambda e: (e["time"], e["segment"], order[e["kind"]], e["position"], e["thread"]))
    return {f: getattr(out, f) for f, _ in _TrialOut._fields_}, events


def run(cfg: Config, seed: int, first: int = 0, count: int = 1, pattern: bool = False,
        per_trial: bool = True, hist: bool = False) -> dict:
    """Trials first..first+count-1 -> exact integer sums (+ per-trial arrays, histograms)."""
    lib = _load()
    sums = _Sums()
    arrs = {}
    ptrs = [None] * 5
    if per_trial:
        for i, (name, dt) in enumerate([("acc", np.int32), ("m", np.int32), ("iters", np.int32),
                                        ("si", np.int64), ("dsi", np.int64)]):
            arrs[name] = np.zeros(count, dt)
            ptrs[i] = arrs[name].ctypes.data
    si_hist = np.zeros(cfg.lookahead + 1, np.int64) if hist else None
    seg_hist = np.zeros(64, np.int64) if hist else None
    rc = lib.oracle_run(ctypes.byref(cfg._c()), seed, first, count, int(pattern),
                        ctypes.byref(sums), *ptrs,
                        si_hist.ctypes.data if hist else None,
                        seg_hist.ctypes.data if hist else None)
    if rc:
        raise ValueError(f"oracle_run failed for {cfg}")
    out = {f: int(getattr(sums, f)) for f, _ in _Sums._fields_}
    out["nonsi"] = (cfg.t_target_first or cfg.t_target) + (cfg.n_tokens - 1) * cfg.t_target
    out.update(arrs)
    if hist:
        out["si_hist"], out["seg_hist"] = si_hist, seg_hist
    return out


def means(sums: dict, tick: float = 1.0) -> dict:
    """FP64 per-config means in user units: ((double)sum / (double)T) * tick."""
    T = float(sums["trials"])
    return {"mean_nonsi": float(sums["nonsi"]) * tick,
            "mean_si": (float(sums["sum_si"]) / T) * tick,
            "mean_dsi": (float(sums["sum_dsi"]) / T) * tick}


def eq1_feasible(t_target: int, t_drafter: int, k: int, sp: int) -> bool:
    """Eq. 1: ceil(t_t / (k t_d)) <= SP, in exact integers."""
    return -(-t_target // (k * t_drafter)) <= sp


def min_lookahead(t_target: int, t_drafter: int, sp: int) -> int:
    """Smallest k >= 1 with ceil(t_t/(k t_d)) <= SP."""
    k = 1
    while not eq1_feasible(t_target, t_drafter, k, sp):
        k += 1
    return k


def required_processors(t_target: int, t_drafter: int, k: int) -> int:
    """1 + ceil(t_t / (k t_d)): one drafter GPU plus the target servers."""
    return 1 + -(-t_target // (k * t_drafter))


# ---- multi-drafter DSI (dsi_oracle_multi.c) ------------------------------
MAX_MODELS = 8


class _MultiConfig(ctypes.Structure):
    _fields_ = [("t_target", ctypes.c_int64), ("t_drafter", ctypes.c_int64 * (MAX_MODELS - 1)),
                ("accept_rate", ctypes.c_double * (MAX_MODELS - 1)),
                ("n_drafters", ctypes.c_int32), ("n_tokens", ctypes.c_int32),
                ("stream_id", ctypes.c_uint32), ("rng_halves", ctypes.c_int32)]


class _MultiOut(ctypes.Structure):
    _fields_ = [("nonsi", ctypes.c_int64), ("dsi", ctypes.c_int64),
                ("settled", ctypes.c_int32 * MAX_MODELS), ("threads", ctypes.c_int64)]


class _MultiSums(ctypes.Structure):
    _fields_ = [("trials", ctypes.c_uint64), ("sum_dsi", ctypes.c_int64),
                ("sumsq_dsi", ctypes.c_uint64), ("sum_settled", ctypes.c_int64 * MAX_MODELS),
                ("n_dsi_gt_nonsi", ctypes.c_int64)]


_multi_ready = False


def _load_multi():
    global _multi_ready
    lib = _load()
    if not _multi_ready:
        P = ctypes.POINTER
        lib.oracle_multi_indicator.argtypes = [P(_MultiConfig), ctypes.c_uint64, ctypes.c_uint64,
                                               ctypes.c_int, ctypes.c_int32, ctypes.c_int32]
        lib.oracle_multi_indicator.restype = ctypes.c_int
        lib.oracle_multi_tree.argtypes = [P(_MultiConfig), ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_int, ctypes.c_int64, P(_MultiOut)]
        lib.oracle_multi_tree.restype = ctypes.c_int
        lib.oracle_multi_chain.argtypes = [P(_MultiConfig), ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_int, P(_MultiOut)]
        lib.oracle_multi_chain.restype = ctypes.c_int
        lib.oracle_multi_run.argtypes = [P(_MultiConfig), ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_int, P(_MultiSums),
                                         ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_multi_run.restype = ctypes.c_int
        _multi_ready = True
    return lib


@dataclass(frozen=True)
class MultiConfig:
    """Algorithm 1 with m = len(t_drafters) + 1 models, lookahead 1, integer ticks.
    Drafters are ordered by latency, t_drafters[0] <= ... <= t_target (R25)."""
    t_target: int
    t_drafters: tuple
    accept_rates: tuple
    n_tokens: int
    stream_id: int = 0
    rng_halves: bool = False  # the halves layout (R26); drafter j on counter word 2(j-1)

    @property
    def m(self) -> int:
        return len(self.t_drafters) + 1

    def _c(self) -> _MultiConfig:
        c = _MultiConfig()
        c.t_target = int(self.t_target)
        for j, (t, a) in enumerate(zip(self.t_drafters, self.accept_rates)):
            c.t_drafter[j] = int(t)
            c.accept_rate[j] = float(a)
        c.n_drafters = len(self.t_drafters)
        c.n_tokens = int(self.n_tokens)
        c.stream_id = int(self.stream_id)
        c.rng_halves = int(bool(self.rng_halves))
        return c


def multi_indicator(cfg: MultiConfig, seed: int, trial: int, j: int, p: int,
                    pattern: bool = False) -> int:
    r = _load_multi().oracle_multi_indicator(ctypes.byref(cfg._c()), seed, trial, int(pattern), j, p)
    if r < 0:
        raise ValueError("oracle_multi_indicator: bad input")
    return int(r)


def _multi_out(o: _MultiOut, m: int) -> dict:
    return {"nonsi": int(o.nonsi), "dsi": int(o.dsi),
            "settled": [int(o.settled[j]) for j in range(m)], "threads": int(o.threads)}


def multi_tree(cfg: MultiConfig, seed: int, trial: int, pattern: bool = False,
               max_threads: int = 1 << 22) -> dict:
    """Literal thread-tree simulation of Algorithm 1 (small N only)."""
    o = _MultiOut()
    rc = _load_multi().oracle_multi_tree(ctypes.byref(cfg._c()), seed, trial, int(pattern),
                                         max_threads, ctypes.byref(o))
    if rc == -2:
        raise OverflowError("oracle_multi_tree: thread budget exceeded")
    if rc:
        raise ValueError(f"oracle_multi_tree failed for {cfg}")
    return _multi_out(o, cfg.m)


def multi_chain(cfg: MultiConfig, seed: int, trial: int, pattern: bool = False) -> dict:
    o = _MultiOut()
    if _load_multi().oracle_multi_chain(ctypes.byref(cfg._c()), seed, trial, int(pattern),
                                        ctypes.byref(o)):
        raise ValueError(f"oracle_multi_chain failed for {cfg}")
    return _multi_out(o, cfg.m)


def multi_run(cfg: MultiConfig, seed: int, first: int = 0, count: int = 1,
              pattern: bool = False, per_trial: bool = True) -> dict:
    """Trials first..first+count-1 (chain simulation) -> exact sums (+ per-trial arrays)."""
    sums = _MultiSums()
    dsi = np.zeros(count, np.int64) if per_trial else None
    settled = np.zeros((count, cfg.m), np.int32) if per_trial else None
    rc = _load_multi().oracle_multi_run(ctypes.byref(cfg._c()), seed, first, count, int(pattern),
                                        ctypes.byref(sums),
                                        dsi.ctypes.data if per_trial else None,
                                        settled.ctypes.data if per_trial else None)
    if rc:
        raise ValueError(f"oracle_multi_run failed for {cfg}")
    out = {"trials": int(sums.trials), "sum_dsi": int(sums.sum_dsi),
           "sumsq_dsi": int(sums.sumsq_dsi),
           "sum_settled": [int(sums.sum_settled[j]) for j in range(cfg.m)],
           "n_dsi_gt_nonsi": int(sums.n_dsi_gt_nonsi), "nonsi": cfg.n_tokens * cfg.t_target}
    if per_trial:
        out["dsi"], out["settled"] = dsi, settled
    return out

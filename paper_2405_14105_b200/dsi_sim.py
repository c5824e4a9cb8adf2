"""Thin ctypes binding of include/dsi_sim.h (argument marshalling only).

Every step of the simulation runs in libdsi_sim.so (sm_100a kernels + C++ host
runtime).  There is no Python or CPU fallback: importing this module without
the built library raises ImportError, and creating a simulator without an
sm_100 GPU fails with DSI_E_DEVICE.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libdsi_sim.so")
# Builds of the same sources (paper_2405_14105_b200/build.py): the product, and two test builds
# that add include/dsi_sim_testing.h (the host all-reduce hook, A/B knobs) -- the second with a
# deliberately wrong C(g) for the mutation test.  The product is what every call uses unless a
# test selects another build with use_library() (or DSI_SIM_LIB=test|mutant|checked|<path> for a whole
# process, e.g. an A/B run).
VARIANT_PATHS = {"product": LIB_PATH, "test": os.path.join(_PKG, "libdsi_sim_test.so"),
                 "mutant": os.path.join(_PKG, "libdsi_sim_mutant.so"),
                 "checked": os.path.join(_PKG, "libdsi_sim_checked.so")}

DSI_ABI_VERSION = 2
DSI_OK, DSI_E_NULL, DSI_E_RANGE, DSI_E_TICK, DSI_E_OVERFLOW, DSI_E_STRICT_EQ1, DSI_E_DEVICE, \
    DSI_E_COMM, DSI_E_STATE, DSI_E_NOMEM = range(10)
DSI_F_PER_TRIAL, DSI_F_HIST, DSI_F_PATTERN, DSI_F_STRICT_EQ1, DSI_F_TIMING = 0x1, 0x2, 0x4, 0x8, 0x10
DSI_F_SHARED_STREAMS = 0x20
DSI_F_FRESH_VERIFIER = 0x40
DSI_F_MEANS_ONLY = 0x80
DSI_F_REDUCE_TO_ROOT = 0x100
DSI_F_RNG_HALVES = 0x200

# Structured dtypes with the exact C layouts (numpy arrays are passed by pointer).
CONFIG_DTYPE = np.dtype([("t_target", "<f8"), ("t_drafter", "<f8"), ("accept_rate", "<f8"),
                         ("lookahead", "<i4"), ("sp_degree", "<i4"), ("n_tokens", "<i4"),
                         ("stream_id", "<u4"), ("n_trials", "<u8"), ("ttft_target", "<f8"),
                         ("ttft_drafter", "<f8")])
RESULT_DTYPE = np.dtype([("trials", "<u8"), ("t_target_ticks", "<i8"), ("t_drafter_ticks", "<i8"),
                         ("nonsi_ticks", "<i8"), ("sum_si_ticks", "<i8"), ("sum_dsi_ticks", "<i8"),
                         ("sumsq_si_ticks", "<u8"), ("sumsq_dsi_ticks", "<u8"),
                         ("sum_si_iters", "<i8"), ("sum_accepts", "<i8"), ("sum_segments", "<i8"),
                         ("n_dsi_gt_nonsi", "<i8"), ("n_dsi_gt_si", "<i8"), ("threshold", "<u8"),
                         ("eq1_feasible", "<i4"), ("min_lookahead", "<i4"),
                         ("mean_nonsi", "<f8"), ("mean_si", "<f8"), ("mean_dsi", "<f8"),
                         ("std_si", "<f8"), ("std_dsi", "<f8")])
HEATMAP_DTYPE = np.dtype([("t_target", "<f8"), ("t_drafter", "<f8"), ("accept_rate", "<f8"),
                          ("sp_degree", "<i4"), ("n_tokens", "<i4"), ("si_lookahead", "<i4"),
                          ("dsi_lookahead", "<i4"), ("nonsi", "<f8"), ("si", "<f8"), ("dsi", "<f8"),
                          ("r_nonsi_si", "<f8"), ("r_si_dsi", "<f8"), ("r_nonsi_dsi", "<f8"),
                          ("r_min_dsi", "<f8"), ("first_cfg", "<u8"), ("n_cfg", "<u8")])
assert CONFIG_DTYPE.itemsize == 64 and RESULT_DTYPE.itemsize == 160 and HEATMAP_DTYPE.itemsize == 112
DSI_MAX_DRAFTERS = 7
MULTI_CONFIG_DTYPE = np.dtype([("t_target", "<f8"), ("t_drafter", "<f8", (DSI_MAX_DRAFTERS,)),
                               ("accept_rate", "<f8", (DSI_MAX_DRAFTERS,)), ("n_drafters", "<i4"),
                               ("n_tokens", "<i4"), ("stream_id", "<u4"), ("reserved", "<u4"),
                               ("n_trials", "<u8")])
MULTI_RESULT_DTYPE = np.dtype([("trials", "<u8"), ("t_target_ticks", "<i8"), ("nonsi_ticks", "<i8"),
                               ("sum_dsi_ticks", "<i8"), ("sumsq_dsi_ticks", "<u8"),
                               ("sum_settled", "<i8", (DSI_MAX_DRAFTERS + 1,)),
                               ("n_dsi_gt_nonsi", "<i8"), ("mean_nonsi", "<f8"), ("mean_dsi", "<f8"),
                               ("std_dsi", "<f8")])
assert MULTI_CONFIG_DTYPE.itemsize == 144 and MULTI_RESULT_DTYPE.itemsize == 136


class dsi_options(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("tick", ctypes.c_double), ("seed", ctypes.c_uint64), ("device", ctypes.c_int32),
                ("n_devices", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("n_shards", ctypes.c_int32),
                ("block_threads", ctypes.c_int32), ("stream", ctypes.c_void_p)]


def _load(path: str):
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, V = ctypes.POINTER, ctypes.c_void_p
    u64, i32, i64, sz = ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    sigs = {
        "dsi_sim_create": ([P(dsi_options), V, sz, P(V)], ctypes.c_int),
        "dsi_sim_update": ([V, V, sz], ctypes.c_int),
        "dsi_sim_run": ([V], ctypes.c_int),
        "dsi_sim_reduce": ([V, V, sz], ctypes.c_int),
        "dsi_sim_trials": ([V, sz, u64, u64, V, V, V, V, V], ctypes.c_int),
        "dsi_sim_hist": ([V, sz, V, V, sz], ctypes.c_int),
        "dsi_sim_stream": ([V, i32, P(V)], ctypes.c_int),
        "dsi_sim_launches": ([V, P(i32)], ctypes.c_int),
        "dsi_sim_kernel_ms": ([V, i32, P(ctypes.c_float)], ctypes.c_int),
        "dsi_sim_reduce_device": ([V], ctypes.c_int),
        "dsi_sim_fetch": ([V, ctypes.c_size_t, ctypes.c_size_t, V], ctypes.c_int),
        "dsi_sim_units": ([V, P(u64), P(u64), P(u64)], ctypes.c_int),
        "dsi_sim_io_bytes": ([V, P(u64), P(u64)], ctypes.c_int),
        "dsi_sim_comm_info": ([V, P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32)],
                              ctypes.c_int),
        "dsi_sim_destroy": ([V], None),
        "dsi_status_str": ([ctypes.c_int], ctypes.c_char_p),
        "dsi_sim_last_error": ([V], ctypes.c_char_p),
        "dsi_last_create_error": ([], ctypes.c_char_p),
        "dsi_abi_version": ([], ctypes.c_uint32),
        "dsi_nccl_unique_id": ([V], ctypes.c_int),
        "dsi_ticks": ([ctypes.c_double, ctypes.c_double, P(ctypes.c_int64)], ctypes.c_int),
        "dsi_min_lookahead": ([i64, i64, i32], i32),
        "dsi_required_processors": ([i64, i64, i32], i32),
        "dsi_eq1_feasible": ([i64, i64, i32, i32], i32),
        "dsi_shard_bounds": ([V, u64, i32, V], ctypes.c_int),
        "dsi_heatmap": ([V, V, sz, V, sz, P(sz)], ctypes.c_int),
        "dsi_sim_heatmap": ([V, V, sz, P(sz)], ctypes.c_int),
        "dsi_heatmap_csv": ([V, sz, ctypes.c_char_p], ctypes.c_int),
        "dsi_multi_simulate": ([P(dsi_options), V, sz, V, V, V], ctypes.c_int),
        "dsi_multi_last_kernel": ([P(ctypes.c_float), P(i32)], ctypes.c_int),
        "dsi_build_id": ([], ctypes.c_char_p),
    }
    testing = {"dsi_set_host_allreduce": ([V, V], ctypes.c_int),
               "dsi_test_set_knob": ([ctypes.c_char_p, i32], ctypes.c_int)}
    for name, (args, res) in list(sigs.items()) + list(testing.items()):
        if name in testing and not hasattr(lib, name):
            continue  # the product build has no test hooks
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


_libs = {}


def load_library(variant: str = "product"):
    """The ctypes handle of one build ("product", "test", "mutant" or a path), loaded once."""
    path = VARIANT_PATHS.get(variant, variant)
    if path not in _libs:
        _libs[path] = _load(path)
    return _libs[path]


lib = load_library(os.environ.get("DSI_SIM_LIB", "product"))


class use_library:
    """Context manager: calls made inside use the given build (handles keep the build they were
    created with).  Tests use it for the test build's hooks and for the mutation test."""

    def __init__(self, variant: str):
        self.variant = variant

    def __enter__(self):
        global lib
        self._prev = lib
        lib = load_library(self.variant)
        return lib

    def __exit__(self, *exc):
        global lib
        lib = self._prev


def select_library(variant: str) -> None:
    """Use another build for the rest of the process (multi-rank test runs on one GPU)."""
    global lib
    lib = load_library(variant)


class _Handle(ctypes.c_void_p):
    """A dsi_sim* that remembers the library build it belongs to."""
    _lib = None


def _L(h):
    return h._lib if isinstance(h, _Handle) and h._lib is not None else lib


def dsi_build_id() -> str:
    """SHA-256 of the sources the loaded product library was built from (dsi_build_id)."""
    return lib.dsi_build_id().decode()
EXPORTED = ("dsi_sim_create", "dsi_sim_update", "dsi_sim_run", "dsi_sim_reduce", "dsi_sim_trials", "dsi_sim_hist",
            "dsi_sim_stream", "dsi_sim_launches", "dsi_sim_kernel_ms", "dsi_sim_units", "dsi_sim_io_bytes", "dsi_sim_reduce_device", "dsi_sim_fetch",
            "dsi_sim_comm_info", "dsi_sim_destroy", "dsi_status_str", "dsi_sim_last_error", "dsi_last_create_error",
            "dsi_abi_version", "dsi_nccl_unique_id", "dsi_ticks", "dsi_min_lookahead",
            "dsi_required_processors", "dsi_eq1_feasible", "dsi_shard_bounds", "dsi_heatmap",
            "dsi_heatmap_csv", "dsi_sim_heatmap", "dsi_multi_simulate", "dsi_multi_last_kernel",
            "dsi_build_id")
TEST_EXPORTED = ("dsi_set_host_allreduce", "dsi_test_set_knob")  # include/dsi_sim_testing.h


class DsiError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        super().__init__(f"{lib.dsi_status_str(status).decode()}{': ' + msg if msg else ''}")


def _check(status: int, handle=None, create: bool = False):
    if status != DSI_OK:
        if create:
            msg = lib.dsi_last_create_error().decode()
        else:
            msg = _L(handle).dsi_sim_last_error(handle).decode() if handle else ""
        raise DsiError(status, msg)


def _testing():
    if not hasattr(lib, "dsi_test_set_knob"):
        raise RuntimeError("test hooks exist only in the test build: wrap the call in use_library('test')")
    return lib


def dsi_test_set_knob(name: str, value: int) -> None:
    """Test build only (include/dsi_sim_testing.h): a launch-planner A/B knob."""
    _check(_testing().dsi_test_set_knob(name.encode(), int(value)))


# ----------------------------------------------------------------------------- same names as the C ABI
def dsi_ticks(x: float, tick: float) -> int:
    """R15: round(x / tick), raising DsiError (DSI_E_RANGE / DSI_E_TICK) like dsi_sim_create."""
    out = ctypes.c_int64()
    _check(lib.dsi_ticks(float(x), float(tick), ctypes.byref(out)))
    return out.value


def dsi_min_lookahead(t_target_ticks: int, t_drafter_ticks: int, sp: int) -> int:
    return lib.dsi_min_lookahead(t_target_ticks, t_drafter_ticks, sp)


def dsi_required_processors(t_target_ticks: int, t_drafter_ticks: int, k: int) -> int:
    return lib.dsi_required_processors(t_target_ticks, t_drafter_ticks, k)


def dsi_eq1_feasible(t_target_ticks: int, t_drafter_ticks: int, k: int, sp: int) -> int:
    return lib.dsi_eq1_feasible(t_target_ticks, t_drafter_ticks, k, sp)


def dsi_shard_bounds(costs, parts: int) -> np.ndarray:
    c = np.ascontiguousarray(costs, dtype=np.float64)
    b = np.zeros(parts + 1, np.uint64)
    _check(lib.dsi_shard_bounds(c.ctypes.data, c.size, parts, b.ctypes.data))
    return b


def dsi_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib.dsi_nccl_unique_id(ctypes.addressof(buf)))
    return bytes(buf)


def dsi_heatmap(configs: np.ndarray, results: np.ndarray) -> np.ndarray:
    """Per-cell argmin over lookaheads and the four ratio panels (Fig. 3 / Fig. 5)."""
    configs = np.ascontiguousarray(configs, dtype=CONFIG_DTYPE)
    results = np.ascontiguousarray(results, dtype=RESULT_DTYPE)
    if configs.size != results.size:
        raise ValueError("configs and results differ in length")
    n = ctypes.c_size_t()
    _check(lib.dsi_heatmap(configs.ctypes.data, results.ctypes.data, configs.size, None, 0, ctypes.byref(n)))
    cells = np.zeros(n.value, HEATMAP_DTYPE)
    _check(lib.dsi_heatmap(configs.ctypes.data, results.ctypes.data, configs.size, cells.ctypes.data,
                           cells.size, ctypes.byref(n)))
    return cells


def dsi_heatmap_csv(cells: np.ndarray, path: str) -> None:
    cells = np.ascontiguousarray(cells, dtype=HEATMAP_DTYPE)
    _check(lib.dsi_heatmap_csv(cells.ctypes.data, cells.size, os.fsencode(path)))


def make_configs(n: int) -> np.ndarray:
    return np.zeros(n, CONFIG_DTYPE)


def make_multi_configs(n: int) -> np.ndarray:
    return np.zeros(n, MULTI_CONFIG_DTYPE)


def dsi_multi_simulate(configs: np.ndarray, *, tick: float, seed: int, flags: int = 0, device: int = 0,
                       stream: int | None = None, per_trial: bool = False, rank: int = 0, world: int = 1,
                       nccl_id: bytes | None = None, n_shards: int = 0) -> tuple:
    """Multi-drafter DSI (Algorithm 1 with m models, lookahead 1) on one device.  Returns
    (results, trial_dsi, trial_settled); the per-trial arrays (config-major, settled with 8
    columns) are None unless per_trial (which adds DSI_F_PER_TRIAL)."""
    configs = np.ascontiguousarray(configs, dtype=MULTI_CONFIG_DTYPE)
    if per_trial:
        flags |= DSI_F_PER_TRIAL
    idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
    opt = dsi_options(DSI_ABI_VERSION, flags, tick, seed, device, 1, rank, world,
                      ctypes.addressof(idbuf) if idbuf is not None else None, n_shards, 0, stream)
    out = np.zeros(configs.size, MULTI_RESULT_DTYPE)
    dsi = settled = None
    if flags & DSI_F_PER_TRIAL:
        total = int(configs["n_trials"].sum())
        dsi = np.zeros(total, np.int32)
        settled = np.zeros((total, 8), np.int32)
    _check(lib.dsi_multi_simulate(ctypes.byref(opt), configs.ctypes.data, configs.size, out.ctypes.data,
                                  dsi.ctypes.data if dsi is not None else None,
                                  settled.ctypes.data if settled is not None else None), create=True)
    return out, dsi, settled


HOST_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t,
                                     ctypes.c_void_p)
_host_allreduce_ref = None  # keeps the ctypes callback alive while registered


def dsi_set_host_allreduce(fn) -> None:
    """Test hook: cross-rank sums through fn(words: np.ndarray[uint64]) -> None, which must sum
    the array element-wise over all ranks in place (e.g. a torch.distributed gloo all_reduce).
    None clears it.  See include/dsi_sim.h."""
    global _host_allreduce_ref
    if fn is None:
        _host_allreduce_ref = None
        _check(_testing().dsi_set_host_allreduce(None, None))
        return

    def cb(buf, n, _user):
        try:
            fn(np.ctypeslib.as_array(buf, shape=(n,)))
            return 0
        except Exception:  # noqa: BLE001  (reported to the library as a failed hook)
            return 1

    _host_allreduce_ref = HOST_ALLREDUCE_FN(cb)
    _check(_testing().dsi_set_host_allreduce(ctypes.cast(_host_allreduce_ref, ctypes.c_void_p), None))


def dsi_multi_last_kernel() -> tuple:
    """(kernel ms of the last dsi_multi_simulate with DSI_F_TIMING, its launches)."""
    ms, n = ctypes.c_float(), ctypes.c_int32()
    _check(lib.dsi_multi_last_kernel(ctypes.byref(ms), ctypes.byref(n)))
    return float(ms.value), int(n.value)


def dsi_sim_create(configs: np.ndarray, *, tick: float, seed: int, flags: int = 0, device: int = 0,
                   n_devices: int = 1, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                   n_shards: int = 0, block_threads: int = 0, stream: int | None = None):
    configs = np.ascontiguousarray(configs, dtype=CONFIG_DTYPE)
    idbuf = None
    if nccl_id is not None:
        idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
    opt = dsi_options(DSI_ABI_VERSION, flags, tick, seed, device, n_devices, rank, world,
                      ctypes.addressof(idbuf) if idbuf is not None else None, n_shards,
                      block_threads, stream)
    h = _Handle()
    _check(lib.dsi_sim_create(ctypes.byref(opt), configs.ctypes.data, configs.size, ctypes.byref(h)),
           create=True)
    h._lib = lib
    return h


def dsi_sim_update(h, configs: np.ndarray) -> None:
    configs = np.ascontiguousarray(configs, dtype=CONFIG_DTYPE)
    _check(_L(h).dsi_sim_update(h, configs.ctypes.data, configs.size), h)


def dsi_sim_run(h) -> None:
    _check(_L(h).dsi_sim_run(h), h)


def dsi_sim_reduce(h, n: int, out: np.ndarray | None = None) -> np.ndarray:
    if out is None:
        out = np.zeros(n, RESULT_DTYPE)
    _check(_L(h).dsi_sim_reduce(h, out.ctypes.data, n), h)
    return out


def dsi_sim_reduce_device(h) -> None:
    _check(_L(h).dsi_sim_reduce_device(h), h)


def dsi_sim_fetch(h, first: int, count: int, out: np.ndarray | None = None) -> np.ndarray:
    if out is None:
        out = np.zeros(count, RESULT_DTYPE)
    assert out.dtype == RESULT_DTYPE and out.size >= count and out.flags["C_CONTIGUOUS"]
    _check(_L(h).dsi_sim_fetch(h, first, count, out.ctypes.data), h)
    return out[:count]


def dsi_sim_heatmap(h, out: np.ndarray | None = None) -> np.ndarray:
    """On-device heatmap product after a run (every rank must call it)."""
    n = ctypes.c_size_t()
    _check(_L(h).dsi_sim_heatmap(h, None, 0, ctypes.byref(n)), h)
    if out is None or out.size != n.value:
        out = np.zeros(n.value, HEATMAP_DTYPE)
    _check(_L(h).dsi_sim_heatmap(h, out.ctypes.data, out.size, ctypes.byref(n)), h)
    return out


def dsi_sim_trials(h, cfg: int, first: int, count: int) -> dict:
    arrs = {k: np.zeros(count, np.int32) for k in ("acc", "m", "iters", "si", "dsi")}
    _check(_L(h).dsi_sim_trials(h, cfg, first, count, *[arrs[k].ctypes.data for k in
                                                      ("acc", "m", "iters", "si", "dsi")]), h)
    return arrs


def dsi_sim_hist(h, cfg: int, k: int) -> tuple:
    seg = np.zeros(64, np.int64)
    si = np.zeros(k + 1, np.int64)
    _check(_L(h).dsi_sim_hist(h, cfg, seg.ctypes.data, si.ctypes.data, k + 1), h)
    return seg, si


def dsi_sim_stream(h, device_index: int = 0) -> int:
    s = ctypes.c_void_p()
    _check(_L(h).dsi_sim_stream(h, device_index, ctypes.byref(s)), h)
    return s.value or 0


def dsi_sim_launches(h) -> int:
    n = ctypes.c_int32()
    _check(_L(h).dsi_sim_launches(h, ctypes.byref(n)), h)
    return n.value


def dsi_sim_kernel_ms(h, device_index: int = 0) -> float:
    ms = ctypes.c_float()
    _check(_L(h).dsi_sim_kernel_ms(h, device_index, ctypes.byref(ms)), h)
    return ms.value


def dsi_sim_units(h) -> tuple:
    a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _check(_L(h).dsi_sim_units(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), h)
    return a.value, b.value, c.value


def dsi_sim_comm_info(h) -> dict:
    """The handle's cross-rank exchange as the communicator reports it (transport: none, nccl, host)."""
    n, r, t, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(_L(h).dsi_sim_comm_info(h, ctypes.byref(n), ctypes.byref(r), ctypes.byref(t), ctypes.byref(c)), h)
    return {"nranks": n.value, "rank": r.value, "transport": ("none", "nccl", "host")[t.value],
            "heatmap_exchange": "cells" if c.value else "moments"}


def dsi_sim_io_bytes(h) -> tuple:
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    _check(_L(h).dsi_sim_io_bytes(h, ctypes.byref(a), ctypes.byref(b)), h)
    return a.value, b.value


def dsi_sim_destroy(h) -> None:
    if h:
        _L(h).dsi_sim_destroy(h)


class Simulator:
    """RAII wrapper: create on construction, destroy on close/exit."""

    def __init__(self, configs: np.ndarray, **kw):
        self.configs = np.ascontiguousarray(configs, dtype=CONFIG_DTYPE)
        self.n = self.configs.size
        self.h = dsi_sim_create(self.configs, **kw)

    def update(self, configs: np.ndarray) -> "Simulator":
        configs = np.ascontiguousarray(configs, dtype=CONFIG_DTYPE)
        dsi_sim_update(self.h, configs)
        self.configs = configs
        return self

    def run(self) -> "Simulator":
        dsi_sim_run(self.h)
        return self

    def reduce(self, out: np.ndarray | None = None) -> np.ndarray:
        """Per-config results; pass a preallocated RESULT_DTYPE array to reuse its pages."""
        return dsi_sim_reduce(self.h, self.n, out)

    def reduce_device(self) -> "Simulator":
        dsi_sim_reduce_device(self.h)
        return self

    def fetch(self, first: int = 0, count: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        return dsi_sim_fetch(self.h, first, self.n - first if count is None else count, out)

    def trials(self, cfg: int, first: int = 0, count: int | None = None) -> dict:
        if count is None:
            count = int(self.configs["n_trials"][cfg]) - first
        return dsi_sim_trials(self.h, cfg, first, count)

    def heatmap(self, out: np.ndarray | None = None) -> np.ndarray:
        """Per-cell argmins and ratio panels computed on the device."""
        return dsi_sim_heatmap(self.h, out)

    def hist(self, cfg: int) -> tuple:
        return dsi_sim_hist(self.h, cfg, int(self.configs["lookahead"][cfg]))

    def kernel_ms(self, device_index: int = 0) -> float:
        return dsi_sim_kernel_ms(self.h, device_index)

    def launches(self) -> int:
        return dsi_sim_launches(self.h)

    def comm_info(self) -> dict:
        return dsi_sim_comm_info(self.h)

    def io_bytes(self) -> tuple:
        return dsi_sim_io_bytes(self.h)

    def stream(self, device_index: int = 0) -> int:
        return dsi_sim_stream(self.h, device_index)

    def close(self) -> None:
        if self.h:
            dsi_sim_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""B200-native Monte Carlo latency simulator of Distributed Speculative Inference (arXiv 2405.14105).

The product is ``libdsi_sim.so`` (C ABI in ``include/dsi_sim.h``: sm_100a trial kernel +
C++ host runtime + NCCL all-reduce).  ``dsi_sim`` is its thin ctypes binding;
``workloads`` builds the seeded synthetic config grids of BASELINE.json.
Attributes of ``dsi_sim`` are re-exported lazily so that ``workloads`` can be
imported without the built library.
"""
import importlib

__all__ = ["dsi_sim", "workloads", "Simulator"]


def __getattr__(name):
    if name == "Simulator" or name.startswith("dsi_sim_") or name.startswith("DSI_"):
        return getattr(importlib.import_module(__name__ + ".dsi_sim"), name)
    raise AttributeError(name)

"""paper_2605_18566_b200 — B200-native Monte-Carlo frozen-coefficient Cole–Hopf solver for
viscous HJ(I) reachability (arxiv/paper_2605_18566), as a C-ABI CUDA library (libhjmc.so,
include/hjmc.h) plus this thin Python binding.

    from paper_2605_18566_b200 import Solver, SolverConfig, inputs
    s = Solver(SolverConfig.from_preset(inputs.C2))
    out = s.solve_slice(inputs.queries(inputs.C2))      # v, dv, c, tube, vhist, chist, g0

The binding loads libhjmc.so lazily on first use and raises if it is missing: there is no
CPU fallback anywhere on the path.
"""
from . import inputs  # noqa: F401  (no arithmetic; safe without the CUDA library)

__all__ = ["Solver", "SolverConfig", "residual_partials", "supported", "inputs", "shard"]


def __getattr__(name):
    import importlib

    if name in ("Solver", "SolverConfig", "residual_partials", "supported"):
        return getattr(importlib.import_module(__name__ + ".solver"), name)
    if name in ("shard", "roofline", "solver", "build"):
        return importlib.import_module(__name__ + "." + name)
    raise AttributeError(name)

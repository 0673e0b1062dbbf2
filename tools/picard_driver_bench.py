"""Algorithm 1 with its stopping test: host-driven loop (hjmc_picard_pass per iterate, host sync
and host ε test) vs the device-resident graph (hjmc_picard_solve). Usage:
  python tools/picard_driver_bench.py [preset-name ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.picard import solve_adaptive, solve_adaptive_device  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402


def timed(f, reps=3):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, r


if __name__ == "__main__":
    names = sys.argv[1:] or ["paper_dubins_40x40", "c2_dubins_n3"]
    for name in names:
        p = I.PRESETS[name]
        s = Solver(SolverConfig.from_preset(p))
        x = torch.from_numpy(I.queries(p)).cuda()
        iters = p.Kp
        th, a = timed(lambda: solve_adaptive(s, x, tol=0.0, max_iter=iters))
        td, b = timed(lambda: solve_adaptive_device(s, x, tol=0.0, max_iter=iters))
        same = all(torch.equal(a[k], b[k]) for k in ("v", "c", "tube"))
        print(json.dumps({"preset": name, "queries": int(x.shape[0]), "K": p.K, "iterates": iters,
                          "host_driven_ms": th, "device_graph_ms": td, "bit_identical": same}))

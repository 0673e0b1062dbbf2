"""The paper's Table 1 setting: the 45-D 14-pursuer / 1-evader game in three speed
regimes, 15 Picard iterations, final relative residual ε(15) — context only: the paper does not
state N, δ, the horizon or the evaluation states (its 7.2 MB per iteration suggests N ≈ 20,000
in double). We run N = 20,000, δ = 0.08, τ = 1, the preset's 32×32 evader slice (1,024 states,
pursuers on a ring of radius 15), CRN, and time Algorithm 1 (host-driven and device graph).
Usage: python tools/table1_multiagent.py"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.picard import solve_adaptive_device  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

PAPER = {"1 evader faster": (1.0, 2.0, 0.003121, 27.6), "2 equal speed": (1.0, 1.0, 0.002454, 30.0),
         "3 pursuers faster": (2.0, 1.0, 0.003462, 27.6)}   # (a_pursuer, a_evader, ε, s)

if __name__ == "__main__":
    for case, (ap, ae, eps_paper, s_paper) in PAPER.items():
        p = I.PAPER_MULTIAGENT45.with_(N=20000, Kp=15, sys_params=(ap, ae))
        s = Solver(SolverConfig.from_preset(p))
        x = torch.from_numpy(I.queries(p)).cuda()
        solve_adaptive_device(s, x, tol=0.0, max_iter=15)          # warm (builds the graph)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = solve_adaptive_device(s, x, tol=0.0, max_iter=15)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"case": case, "a_pursuer": ap, "a_evader": ae, "N": p.N,
                          "states": int(x.shape[0]), "eps15": round(float(r["eps"][0, 14]), 6),
                          "paper_eps": eps_paper, "seconds_1_B200": round(dt, 4),
                          "paper_seconds_16_core_cpu": s_paper}))

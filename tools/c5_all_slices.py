"""BASELINE config 5 as a whole on one B200: all 8 slices (θ₁ = kπ/4) of 256² queries, each with
the exact shortcuts (stationary skip + pass memo + speculative clamps; bit-identical to the full
schedule), and the
full schedule on two of them — the 1-GPU point of the 1/2/4/8-GPU query-sharded run (one slice
per GPU at 8 GPUs). Usage: python tools/c5_all_slices.py [--full 0,4]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402


def timed(solver, x, qid):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = solver.alloc_result(x.shape[0], hist=False)
    solver.pass_count()
    e0.record()
    solver.solve_slice(x, qid=qid, out=out)
    e1.record()
    torch.cuda.synchronize()
    solver.check()
    return e0.elapsed_time(e1) / 1e3, solver.pass_count(), out


if __name__ == "__main__":
    full = ([int(a) for a in sys.argv[sys.argv.index("--full") + 1].split(",") if a]
            if "--full" in sys.argv else [0, 4])
    p = I.C5
    per = p.grid_pts * p.grid_pts
    x_all = torch.from_numpy(I.queries(p)).cuda()
    fast = Solver(SolverConfig.from_preset(p, skip_stationary=True, reuse_passes=True,
                                           speculate=True))
    base = Solver(SolverConfig.from_preset(p))
    fast.solve_slice(x_all[:296])                               # warm both kernels
    base.solve_slice(x_all[:296])
    torch.cuda.synchronize()
    rows, total_fast = [], 0.0
    for k in range(len(p.slices)):
        ids = torch.arange(k * per, (k + 1) * per, dtype=torch.int32, device="cuda")
        x = x_all[k * per:(k + 1) * per]
        t, passes, out = timed(fast, x, ids)
        total_fast += t
        row = {"slice": k, "theta1": round(k * np.pi / 4, 4), "fast_s": round(t, 2),
               "passes_frac": round(passes / (per * p.K * p.Kp), 4),
               "brt_points": int((out["tube"] <= 0).sum())}
        if k in full:
            tf, _, outf = timed(base, x, ids)
            row["full_s"] = round(tf, 2)
            row["bit_identical"] = bool(torch.equal(out["v"], outf["v"]) and torch.equal(out["tube"], outf["tube"]))
        rows.append(row)
        print(json.dumps(row), flush=True)
    full_rows = [r for r in rows if "full_s" in r]
    print(json.dumps({"config": p.name, "slices": len(p.slices), "queries": p.M,
                      "total_fast_s_1gpu": round(total_fast, 1),
                      "full_schedule_slices_measured": len(full_rows),
                      "total_full_s_1gpu": round(sum(r["full_s"] for r in full_rows), 1),
                      "evals_per_s_full": (len(full_rows) * per * p.N * p.K * p.Kp
                                           / max(sum(r["full_s"] for r in full_rows), 1e-9)),
                      "all_bit_identical": all(r["bit_identical"] for r in full_rows),
                      "evals_full_schedule": p.M * p.N * p.K * p.Kp}))

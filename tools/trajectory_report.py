"""Per-query Picard trajectories (c^(k), v^(k) per horizon), GPU vs oracle, for the sampled
full-size C2 queries the parity test uses; prints the queries with the largest v deviation.
Diagnostic only (the oracle is test infrastructure)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from _parity import v_violations  # noqa: E402
from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

p = I.C2
s = Solver(SolverConfig.from_preset(p))
x = I.queries(p)
out = {k: t.cpu().numpy() for k, t in s.solve_slice(x).items()}
spread = I.subsample_ids(x.shape[0], 24)
boundary = np.argsort(np.abs(out["v"]))[:12]
interior = np.flatnonzero((out["chist"][-1, -1] > p.c_min * 1.01) & (out["chist"][-1, -1] < p.c_max * 0.99))[:12]
ids = np.unique(np.concatenate([spread, boundary, interior])).astype(np.int64)
ref = O.solve_slice(O.Problem.from_preset(p), x[ids], qids=ids.astype(np.uint32))
worst = []
for q in range(len(ids)):
    r = max(v_violations(out["vhist"][j, k, ids], ref["vhist"][j, k])[q] for j in range(p.K) for k in range(p.Kp))
    worst.append(r)
order = np.argsort(worst)[::-1][:3]
for q in order:
    m = ids[q]
    print(f"query {m} x={x[m]} worst v ratio {worst[q]:.3f}")
    for j in range(p.K):
        cg = out["chist"][j, :, m]
        co = ref["chist"][j, :, q]
        vg = out["vhist"][j, :, m]
        vo = ref["vhist"][j, :, q]
        if np.max(np.abs(vg - vo) / np.maximum(np.abs(vo), 1e-9)) > 5e-5:
            print(f"  j={j} c_gpu={np.round(cg, 4)}\n       c_orc={np.round(co, 4)}\n       dv_rel={np.array2string((vg - vo) / np.abs(vo), precision=2)}")

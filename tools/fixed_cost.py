"""Per-pass fixed cost of a config's solve kernel: time the same queries at N and N/2 (and N/4);
T(N) = a + b·N per pass, so a is the reduction/barrier/epilogue cost a pass pays regardless of
its samples. Usage: python tools/fixed_cost.py [c5] [queries]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

idx = int(sys.argv[1].lstrip("c")) if len(sys.argv) > 1 else 5
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1184
p0 = I.BY_INDEX[idx]
ids = I.bench_ids(p0)
ids = ids[np.linspace(0, len(ids) - 1, min(nq, len(ids))).round().astype(int)]
x = torch.from_numpy(np.ascontiguousarray(I.queries(p0)[ids])).cuda()
q = torch.from_numpy(ids.astype(np.int32)).cuda()
rows = []
for div in (1, 2, 4):
    p = p0.with_(N=p0.N // div)
    s = Solver(SolverConfig.from_preset(p))
    s.solve_slice(x, qid=q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.solve_slice(x, qid=q)
    e1.record()
    torch.cuda.synchronize()
    rows.append((p.N, e0.elapsed_time(e1)))
(n1, t1), (n2, t2) = rows[0], rows[1]
b = (t1 - t2) / (n1 - n2)
a = t1 - b * n1
print(json.dumps({"config": p0.name, "queries": int(len(ids)), "runs_ms": rows,
                  "fixed_ms_total": a, "fixed_share_at_full_N": a / t1}))

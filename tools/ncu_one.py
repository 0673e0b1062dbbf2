"""One solve_slice launch of a BASELINE config on a query subset with reduced K and Kp, for an
attributable ncu capture of that config's solve kernel ("use a reduced K = Kp = 1
variant of the same kernel"). Usage:
  ncu --set full --clock-control none -k regex:solve_kernel -c 1 -o out \
      python tools/ncu_one.py c5 [queries] [K] [Kp]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import _lib, inputs as I  # noqa: E402

if "--lib" in sys.argv:               # a build variant (tools/build_variants.py)
    i = sys.argv.index("--lib")
    _lib.load(sys.argv[i + 1])
    del sys.argv[i:i + 2]
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

if __name__ == "__main__":
    idx = int(sys.argv[1].lstrip("c")) if len(sys.argv) > 1 else 5
    nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1184
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    Kp = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    p = I.BY_INDEX[idx].with_(K=K, Kp=Kp)
    x_all = I.queries(I.BY_INDEX[idx])
    ids = I.bench_ids(I.BY_INDEX[idx])          # the benchmark's queries (C5: its subset)
    ids = ids[np.linspace(0, len(ids) - 1, min(nq, len(ids))).round().astype(int)]
    s = Solver(SolverConfig.from_preset(p))
    x = torch.from_numpy(x_all[ids]).cuda()
    qid = torch.from_numpy(ids.astype(np.int32)).cuda()
    s.solve_slice(x, qid=qid)
    torch.cuda.synchronize()
    s.check()
    print(f"{p.name}: {nq} queries, K={K}, Kp={Kp}, N={p.N}")

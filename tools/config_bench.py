"""Throughput of solve_slice per BASELINE config on a deterministic query subset (global query
ids kept, so each query's result equals the full launch's). Reports evals/s and the fraction of
the measured-pipe roofline. Usage: python tools/config_bench.py [c3 c4 c5 ...] [--lib path]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import _lib, inputs as I, roofline as RL  # noqa: E402

if "--lib" in sys.argv:
    _lib.load(sys.argv[sys.argv.index("--lib") + 1])
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

SUBSET = {1: None, 2: None, 3: 4096, 4: 2048, 5: 1184}


def run(idx, full_slice=False):
    p = I.BY_INDEX[idx] if isinstance(idx, int) else I.PRESETS[idx]
    x_all = I.queries(p)
    sub = SUBSET.get(idx)
    if full_slice:      # one complete 2-D slice (the first), measured rather than extrapolated
        sub = None
        x_all = x_all[: p.grid_pts * p.grid_pts]
    ids = np.arange(x_all.shape[0]) if sub is None else I.subsample_ids(x_all.shape[0], sub)
    s = Solver(SolverConfig.from_preset(p))
    x = torch.from_numpy(x_all[ids]).cuda()
    qid = torch.from_numpy(ids.astype(np.int32)).cuda()
    out = s.alloc_result(len(ids), hist=False)
    # warm up with the launch actually timed (the kernel variant depends on M·K and N: lazy
    # module loading would otherwise land in the timed region) unless that launch is long
    warm = len(ids) if len(ids) * p.N * p.K * p.Kp < 2e11 else min(len(ids), 296)
    s.solve_slice(x[:warm], qid=qid[:warm])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.solve_slice(x, qid=qid, out=out)
    e1.record()
    torch.cuda.synchronize()
    s.check()
    ms = e0.elapsed_time(e1)
    evals = len(ids) * p.N * p.K * p.Kp
    rl = RL.roofline(p.n, p.target)
    # the same subset with the exact shortcuts (bit-identical outputs): stationary skip + memo
    f = Solver(SolverConfig.from_preset(p, skip_stationary=True, reuse_passes=True, speculate=True))
    fout = f.alloc_result(len(ids), hist=False)
    f.solve_slice(x[:warm], qid=qid[:warm])
    torch.cuda.synchronize()
    f.pass_count()
    e0.record()
    f.solve_slice(x, qid=qid, out=fout)
    e1.record()
    torch.cuda.synchronize()
    fms = e0.elapsed_time(e1)
    fpasses = f.pass_count()
    assert torch.equal(out["v"], fout["v"]) and torch.equal(out["tube"], fout["tube"])
    r = {"config": p.name, "queries": int(len(ids)), "ms": ms, "evals_per_s": evals / (ms / 1e3),
         "frac_of_roofline": evals / (ms / 1e3) / rl["peak_evals_per_s"], "binding": rl["binding_pipe"],
         "full_slice_s_extrapolated": p.M * p.N * p.K * p.Kp / (evals / (ms / 1e3)) / len(p.slices),
         "measured_full_slice": bool(full_slice),
         "fastpath": {"ms": fms, "passes_frac": fpasses / (len(ids) * p.K * p.Kp),
                      "full_slice_s_extrapolated": ms and fms / ms * p.M * p.N * p.K * p.Kp
                      / (evals / (ms / 1e3)) / len(p.slices)}}
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    which = [int(a.lstrip("c")) if a[1:].isdigit() else a
             for a in sys.argv[1:] if (a.startswith("c") and a[1:].isdigit()) or a in I.PRESETS]
    which = which or [2, 3, 4, 5]
    for i in which:
        run(i, full_slice="--full-slice" in sys.argv)

"""GPU-vs-oracle parity report (diagnostic; prints worst ratios to the R20 tolerances for every
quantity and iterate). Usage: python tools/parity_report.py [--full]"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from _parity import c_violations, dv_violations, v_violations  # noqa: E402
from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402


def report(name, preset, x, qids=None):
    s = Solver(SolverConfig.from_preset(preset))
    out = s.solve_slice(x)
    if qids is None:
        ref = O.solve_slice(O.Problem.from_preset(preset), x)
    else:
        out = {k: (t[..., qids] if k in ("vhist", "chist") else t[qids]) for k, t in out.items()}
        ref = O.solve_slice(O.Problem.from_preset(preset), x[qids], qids=qids.astype(np.uint32))
    g = {k: t.cpu().numpy() for k, t in out.items()}
    K, Kp = preset.K, preset.Kp
    vr = max(v_violations(g["vhist"][j, k], ref["vhist"][j, k]).max() for j in range(K) for k in range(Kp))
    cr = max(v_violations(g["chist"][j, k], ref["chist"][j, k]).max() for j in range(K) for k in range(Kp))
    crel = max(np.abs(g["chist"][j, k] / ref["chist"][j, k] - 1).max() for j in range(K) for k in range(Kp))
    P = O.Problem.from_preset(preset)
    xs = x if qids is None else x[qids]
    dg = np.stack([O.dg(P, xm.astype(np.float64)) for xm in xs])
    cb = max(c_violations(O, P, xs, g["chist"][j, k], ref["chist"][j, k],
                          dg if k == 0 else ref["dvhist"][j, k - 1]).max()
             for j in range(K) for k in range(Kp))
    interior = ((ref["chist"] > preset.c_min * 1.001) & (ref["chist"] < preset.c_max * 0.999)).mean()
    print(f"{name:28s} M={x.shape[0] if qids is None else len(qids):6d} "
          f"vhist {vr:7.3f}  v {v_violations(g['v'], ref['v']).max():7.3f}  "
          f"dv {dv_violations(g['dv'], ref['dv']).max():7.3f}  tube {v_violations(g['tube'], ref['tube']).max():7.3f}  "
          f"| chist {cr:7.3f} (max rel {crel:.2e}, interior frac {interior:.3f}; perturbation-bound ratio {cb:.3f})", flush=True)


def grid(lo, hi, pts, fixed):
    a = np.linspace(lo, hi, pts)
    X, Y = np.meshgrid(a, a, indexing="ij")
    x = np.tile(np.asarray(fixed, np.float64), (X.size, 1))
    x[:, 0], x[:, 1] = X.ravel(), Y.ravel()
    return x.astype(np.float32)


if __name__ == "__main__":
    report("dubins small K3Kp4 N3001", I.C2.with_(K=3, Kp=4, N=3001), grid(-20, 20, 11, (0, 0, math.pi / 2)))
    report("rocket6 small", I.C3.with_(K=2, Kp=3, N=2500), grid(-20, 20, 7, (0,) * 6))
    report("pairs5 small", I.C4.with_(K=2, Kp=3, N=1200), grid(-20, 20, 5, I.pair_fixed(5, math.pi / 2)))
    if "--full" in sys.argv:
        x = I.queries(I.C2)
        ids = I.subsample_ids(x.shape[0], 40)
        report("C2 FULL (sampled)", I.C2, x, ids)

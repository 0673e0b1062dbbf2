"""How much of the GPU–oracle difference is the problem's own conditioning? (SURVEY §7 "run the
oracle also in float to measure the intrinsic conditioning"; readings R25/R27.)

For the sampled full-size queries of each config (C2: an even spread of 256 ids, oracle run
here; C3–C5: tests/golden/), compare
  (a) GPU vs oracle:            |v_gpu(x) − v_oracle(x)|,
  (b) GPU vs GPU at x ± 1 ulp:  |v_gpu(x) − v_gpu(nextafter(x))|  (same samples, same kernel),
both in units of the R20 tolerance, at every horizon's final iterate. If (a) is of the order of
(b), the remaining GPU–oracle difference is what a one-ulp change of the fp32 input already
produces — the map's own sensitivity (non-contractive Picard band, R27), not an error of the
kernel. JSON on stdout. Usage: python tools/conditioning_report.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from _parity import FLOOR, V_RTOL  # noqa: E402
from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402


def ratios(a, b, floor):
    return np.abs(a - b) / (V_RTOL * np.maximum(np.abs(b), floor))


def main():
    rows = []
    for idx in (2, 3, 4, 5):
        p = I.BY_INDEX[idx]
        if idx == 2:
            x_all = I.queries(p)
            ids = I.subsample_ids(x_all.shape[0], 256)
            x = x_all[ids]
            ref = O.solve_slice(O.Problem.from_preset(p), x, qids=ids.astype(np.uint32))
            vref = ref["vhist"][:, -1, :]
        else:
            d = np.load(os.path.join(ROOT, "tests", "golden", f"{p.name}_sample.npz"))
            ids, x, vref = d["ids"], d["x"], d["vhist"][:, -1, :]
        s = Solver(SolverConfig.from_preset(p))
        q = ids.astype(np.int32)
        va = s.solve_slice(x, qid=q)["vhist"][:, -1, :].cpu().numpy().astype(np.float64)
        xp = np.nextafter(x, np.float32(np.inf), dtype=np.float32)   # every coordinate + 1 ulp
        vb = s.solve_slice(xp, qid=q)["vhist"][:, -1, :].cpu().numpy().astype(np.float64)
        floor = FLOOR * np.abs(vref).max()
        ra, rb = ratios(va, vref, floor), ratios(vb, va, floor)
        rows.append({"config": p.name, "queries": int(len(ids)), "horizons": p.K,
                     "gpu_vs_oracle": {"median": float(np.median(ra)), "p99": float(np.quantile(ra, 0.99)),
                                       "max": float(ra.max())},
                     "gpu_vs_gpu_1ulp_input": {"median": float(np.median(rb)),
                                               "p99": float(np.quantile(rb, 0.99)),
                                               "max": float(rb.max())}})
    print(json.dumps({"unit": "R20 tolerance on v (1 = at the tolerance)", "rows": rows}))


if __name__ == "__main__":
    main()

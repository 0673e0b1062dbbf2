"""Theorem 1's O(N^-1/2) concentration measured on the GPU: R = 32,768
independent Philox streams (distinct global query ids at one state of the quadratic bowl,
c = 20, τ = 0.5, δ = 0.05), for N = 2^8 … 2^16 samples per estimate. Reports the spread of v̂
against the delta-method standard error CV/(c√N), the mean against the closed form plus its
O(1/N) bias, and the log-log slope of the spread in N (theory: −1/2). JSON on stdout.
Usage: python tools/concentration_report.py"""
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

R = 32768


def main():
    x, c, tau, delta = np.array([0.3, -0.2]), 20.0, 0.5, 0.05
    k = c * delta * tau
    v_true = x @ x / (2 * (1 + k)) - 0.25 + 2 / (2 * c) * math.log1p(k)
    cv2 = ((1 + k) ** 2 / (1 + 2 * k)) * math.exp(c * (x @ x) * (1 / (1 + k) - 1 / (1 + 2 * k))) - 1
    rows, Ns, sds = [], [], []
    for e in range(8, 17, 2):
        N = 1 << e
        s = Solver(SolverConfig(n=2, delta=delta, N=N, seed=0xC0FFEE, system="quadratic",
                                target="quad_bowl", tgt_params=(0.25,)))
        xs = np.tile(x.astype(np.float32), (R, 1))
        v, _ = s.value_grad(xs, np.full(R, c, np.float32), tau, j_tag=9, k_tag=0)
        v = v.cpu().numpy().astype(np.float64)
        se = math.sqrt(cv2 / N) / c
        bias = cv2 / (2 * c * N)
        rows.append({"N": N, "mean": v.mean(), "closed_form_plus_bias": v_true + bias,
                     "mean_error_in_SEs": (v.mean() - v_true - bias) / (se / math.sqrt(R)),
                     "std": v.std(ddof=1), "delta_method_se": se,
                     "std_over_se": v.std(ddof=1) / se})
        Ns.append(N)
        sds.append(v.std(ddof=1))
    slope = float(np.polyfit(np.log(Ns), np.log(sds), 1)[0])
    print(json.dumps({"streams": R, "state": x.tolist(), "c": c, "tau": tau, "delta": delta,
                      "closed_form_v": v_true, "loglog_slope_std_vs_N": slope, "theory": -0.5,
                      "rows": rows}))


if __name__ == "__main__":
    main()

"""Parity of a COMPLETE C2 slice (every query, every horizon, every Picard iterate) between the
CUDA path and the CPU oracle, with the acceptance rules of tests/_parity.py: R20 tolerances on
vhist / v / Dv / tube, the R25 first-order bound on chist, and for a (query, horizon) that fails
those, the R27 bound propagated along the oracle's own trajectory. Reports counts instead of
stopping at the first violation. The oracle needs ≈ 5e10 evaluations (≈ 15 min on 16 cores).
Usage: python tools/full_slice_parity.py [c2] > report.json"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from _parity import (FLOOR, V_RTOL, c_violations, dv_violations, propagated_bounds,  # noqa: E402
                     v_violations)
from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402


def main(name="c2"):
    p = I.BY_INDEX[int(name.lstrip("c"))]
    x = I.queries(p)
    M = x.shape[0]
    t0 = time.time()
    s = Solver(SolverConfig.from_preset(p))
    out = {k: t.cpu().numpy() for k, t in s.solve_slice(x).items()}
    s.check()
    t_gpu = time.time() - t0
    P = O.Problem.from_preset(p)
    t0 = time.time()
    ref = O.solve_slice(P, x)
    t_orc = time.time() - t0
    assert ref["status"] == 0
    xd = x.astype(np.float64)
    floor = FLOOR * np.abs(ref["vhist"]).max()
    dg = np.stack([O.dg(P, xm) for xm in xd])
    plain_ok, propagated_ok, failed, worst_plain = 0, 0, [], 0.0
    for m in range(M):
        for j in range(p.K):
            ok = True
            for k in range(p.Kp):
                vr = ref["vhist"][j, k, m]
                r = abs(out["vhist"][j, k, m] - vr) / (V_RTOL * max(abs(vr), floor))
                p_ref = dg[m] if k == 0 else ref["dvhist"][j, k - 1, m]
                rc = c_violations(O, P, xd[m:m + 1], [out["chist"][j, k, m]],
                                  [ref["chist"][j, k, m]], p_ref[None])[0]
                if r > 1.0 or rc > 1.0:
                    ok = False
                    break
                worst_plain = max(worst_plain, r)
            if ok:
                plain_ok += 1
                continue
            bv, bc, _ = propagated_bounds(O, P, xd[m], m, j + 1, ref["chist"][j, :, m],
                                          ref["vhist"][j, :, m], ref["dvhist"][j, :, m], floor)
            dv = np.abs(out["vhist"][j, :, m] - ref["vhist"][j, :, m])
            dc = np.abs(out["chist"][j, :, m] - ref["chist"][j, :, m])
            if np.all(dv <= bv) and np.all(dc <= bc):
                propagated_ok += 1
            else:
                failed.append([int(m), int(j)])
    # final outputs (v, Dv, tube at τ_K) as tests/test_gpu_parity.py::_final_outputs_within:
    # R20, else the propagated bound of the last horizon's trajectory
    okv = v_violations(out["v"], ref["v"]) <= 1.0
    okd = dv_violations(out["dv"], ref["dv"]) <= 1.0
    okt = v_violations(out["tube"], ref["tube"]) <= 1.0
    final_plain = int(np.sum(okv & okd & okt))
    final_prop, final_failed = 0, []
    for m in np.flatnonzero(~(okv & okd & okt)):
        bv, _, bd = propagated_bounds(O, P, xd[m], m, p.K, ref["chist"][-1, :, m],
                                      ref["vhist"][-1, :, m], ref["dvhist"][-1, :, m], floor)
        if (abs(out["v"][m] - ref["v"][m]) <= bv[-1]
                and np.linalg.norm(out["dv"][m] - ref["dv"][m]) <= bd[-1]):
            final_prop += 1
        else:
            final_failed.append(int(m))
    if os.environ.get("HJMC_PARITY_DUMP"):
        np.savez_compressed(os.environ["HJMC_PARITY_DUMP"], **{f"gpu_{k}": v for k, v in out.items()},
                            **{f"ref_{k}": v for k, v in ref.items() if k != "status"})
    last = (np.abs(ref["chist"][-1, -1] - out["chist"][-1, -1]) > 0)
    rep = {
        "config": p.name, "queries": M, "units": M * p.K, "iterates_per_unit": p.Kp,
        "gpu_s": round(t_gpu, 3), "oracle_s": round(t_orc, 1), "oracle_threads": O.max_threads(),
        "units_within_plain_tolerances": plain_ok,
        "units_within_propagated_bound": propagated_ok,
        "units_failed": len(failed), "failed": failed[:20],
        "worst_vhist_ratio_plain_units": round(float(worst_plain), 4),
        "final_outputs_within_plain_tolerances": final_plain,
        "final_outputs_within_propagated_bound": final_prop,
        "final_outputs_failed": final_failed[:20],
        "worst_ratio_final": {
            "v": round(float(v_violations(out["v"], ref["v"]).max()), 4),
            "dv": round(float(dv_violations(out["dv"], ref["dv"]).max()), 4),
            "tube": round(float(v_violations(out["tube"], ref["tube"]).max()), 4)},
        "g0_max_abs": float(np.abs(out["g0"] - ref["g0"]).max()),
        "final_c_differs_frac": float(last.mean()),
        "tolerances": "R20: |Δv| ≤ 2e-4·max(|v|, 1e-2‖v‖∞), ‖ΔDv‖ ≤ 1e-3·max(‖Dv‖, 1e-2 max‖Dv‖); "
                      "R25 chist bound; R27 propagated bound for non-contractive units",
    }
    print(json.dumps(rep))


if __name__ == "__main__":
    main(*(a for a in sys.argv[1:2]))

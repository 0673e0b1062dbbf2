"""Algorithmic operation counts per query·sample evaluation and the B200 ALU roofline.

The path is bound by plain ALU/MUFU arithmetic (no contraction, ~0 HBM traffic),
so its roofline is a pipe roofline. Per eval the METHOD needs (independent of how the kernel
is written; DESIGN.md §6 derives each line):
  * Philox4x32-10, one call per 4 normals: 10 rounds × (2 wide multiplies + 2 three-input XORs);
    in the first two rounds counter words 1–3 are the same for every sample, leaving
    18 multiplies and 19 XORs per call that depend on the sample index;
  * uniform mapping: one AND/OR + one add per 32-bit word used;
  * Box–Muller: per radius word LG2 + SQRT + 1 multiply; per angle word 1 multiply, COS (+ SIN
    when the second normal of the pair is used) and 1 multiply per normal produced;
  * y = x + σ z on the coordinates g reads, g itself, a = A·core + B (1 FFMA), 1 EX2;
  * the moment update: 1 add + n FFMAs.
Pipe rates (lane-ops per clock per SM) default to the nominal sm_100 figures and are replaced
by the box-measured ones in profiles/pipe_rates.json when present.
"""
from __future__ import annotations

import json
import math
import os

NSM = 148
F_MAX_MHZ = 1965.0

# nominal lane-op rates per SM per clock (4 SMSPs): issue 4×32; FP32 FMA 128; INT multiply
# (IMAD on the FMA-heavy half) 64; logic/ALU 64; MUFU (XU) 16
NOMINAL_RATES = {"issue": 128.0, "fp32": 128.0, "imul": 64.0, "alu": 64.0, "mufu": 16.0}

def op_counts(n: int, target: str, antithetic: bool = False) -> dict:
    """Minimal lane-operation counts per eval, by pipe class (antithetic: one draw of n
    normals serves two samples, so the draw costs are halved)."""
    quads = (n + 3) // 4
    pairs_used = (n + 1) // 2               # Box–Muller pairs with ≥1 normal used
    sins = n // 2                           # second normal of a pair used
    words = 2 * pairs_used
    # ---- per draw: Philox + uniform mapping + Box–Muller
    draw = {"imul": 18 * quads, "alu": 19 * quads + words + 1,
            "fp32": words + 2 * pairs_used + n, "mufu": 3 * pairs_used + sins}
    # ---- per sample: y, g, weight, moments
    samp = {"imul": 0, "alu": 0, "fp32": 0, "mufu": 1}   # EX2
    if target == "quad_bowl":
        samp["fp32"] += 2 * n + 1
    elif target == "linear":
        samp["fp32"] += 2 * n
    elif target == "pair_union":
        K = n // 3
        samp["fp32"] += 4 * K
        samp["alu"] += K
        samp["mufu"] += 1
    elif target == "disk":
        samp["fp32"] += 4
        samp["mufu"] += 1
    elif target == "rel_disk6":
        samp["fp32"] += 8
        samp["mufu"] += 1
    samp["fp32"] += 1 + 1 + n               # a = A·core + B; S += w; M += w z
    f = 0.5 if antithetic else 1.0
    ops = {k: f * draw[k] + samp[k] for k in draw}
    ops["issue"] = sum(ops.values())
    return ops


def load_rates(path: str | None = None) -> tuple[dict, str]:
    path = path or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "profiles", "pipe_rates.json")
    rates = dict(NOMINAL_RATES)
    src = "nominal sm_100 pipe rates"
    if os.path.exists(path):
        with open(path) as fh:
            meas = json.load(fh)
        for k in rates:
            if k in meas.get("lane_ops_per_clk_per_sm", {}):
                rates[k] = float(meas["lane_ops_per_clk_per_sm"][k])
        src = f"measured ({os.path.relpath(path)})"
    return rates, src


def roofline(n: int, target: str, antithetic: bool = False, f_mhz: float = F_MAX_MHZ,
             rates: dict | None = None) -> dict:
    """Evals/s at the binding pipe, and which pipe binds."""
    rates = rates or load_rates()[0]
    ops = op_counts(n, target, antithetic)
    cyc = {k: ops[k] / rates[k] for k in ops}            # SM-clocks per eval per SM
    bound = max(cyc, key=cyc.get)
    evals_per_s = NSM * f_mhz * 1e6 / cyc[bound]
    return {"ops": ops, "cycles_per_eval_per_sm": cyc, "binding_pipe": bound,
            "peak_evals_per_s": evals_per_s, "rate": rates[bound],
            "peak_ops_per_s": rates[bound] * NSM * f_mhz * 1e6}

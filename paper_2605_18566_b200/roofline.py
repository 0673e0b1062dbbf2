"""Algorithmic operation counts per query·sample evaluation and the B200 ALU roofline.

The path is bound by plain ALU/MUFU arithmetic (no contraction, ~0 HBM traffic),
so its roofline is a pipe roofline. Per eval the METHOD needs (independent of how the kernel
is written; DESIGN.md §6 derives each line):
  * Philox4x32-10, one call (block) per 4 normals (draw layout R19 wastes none for n = 2, 3,
    6): 10 rounds × (2 wide multiplies + 2 three-input XORs). Under the counter contract
    (c0 = draw group g, c1 = block | kw<<8 | jw<<16, c2 = query id, c3 = tag) the values that
    depend on neither g nor the block are per-unit constants, and those that depend on g but
    not on the block are shared by the Q blocks of a group. Tracing the rounds:
      multiplies: R1 (g·M0 shared, qid·M1 constant), R2 (b-only: constant; g-only: shared),
                  R3 (one shared, one per block), R4–R10 (2 per block) → 3 per group + 15 per block;
      XORs:       R1 (one b-only constant, one shared), R2 (one shared, one per block),
                  R3–R10 (2 per block)                                → 2 per group + 17 per block;
    the minimum any kernel honouring the contract must execute (the C2 kernel's SASS has
    exactly 48 IMAD.WIDE and 53 XOR-LOP3 per 3-block group);
  * Box–Muller per pair: 2 mantissa builds, 1 add, LG2 + SQRT + COS + SIN, 2 multiplies
    (distance targets — disk, rel-disk-6, pair union, pursuit-min — instead one w·r̂ per
    (sample, pair) in σ-scaled coordinates);
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

def draw_layout(n: int) -> tuple[int, int]:
    """(G, Q): draws per group and Philox blocks per group (R19, include/hjmc.h)."""
    g0 = 1 if n % 4 == 0 else (2 if n % 2 == 0 else 4)
    G = g0 if g0 * n <= 16 else 1
    Q = (n + 3) // 4 if G == 1 else G * n // 4
    return G, Q


def op_counts(n: int, target: str, antithetic: bool = False) -> dict:
    """Minimal lane-operation counts per eval, by pipe class (antithetic: one draw of n
    normals serves two samples, so the draw costs are halved).

    Per draw group (grouped layout): Q Philox blocks, 3 + 15Q wide multiplies and 2 + 17Q
    XORs (module docstring); per Box–Muller pair 2 mantissa builds (ALU), u = F − (1 − 2⁻²⁴)
    and r̂·cos, r̂·sin (3 FP32), LG2 + SQRT + COS + SIN (4 MUFU; the angle a is already in
    revolutions, the MUFU unit's native unit); a pair whose second normal is unused drops its
    SIN and one multiply. Divided by the G draws of the group."""
    G, Q = draw_layout(n)
    used = G * n                                # normals used per group
    pairs = (used + 1) // 2
    half = used % 2                             # a last pair with only its cos used
    # targets whose core is a distance (homogeneous of degree 1 in the position: disk,
    # rel-disk-6, pair union, pursuit-min) need no r̂·cos / r̂·sin products: in σ-scaled
    # coordinates a sample coordinate is one FFMA x/σ' + r̂·trig (counted with the target below)
    # and the moments take w·r̂ once per (sample, pair) the sample touches
    homog = target in ("pair_union", "pursuit_min", "disk", "rel_disk6")
    if homog:
        touched = sum((r * n + n - 1) // 2 - (r * n) // 2 + 1 for r in range(G))
        fp32_draw = pairs + touched
    else:
        fp32_draw = 3 * pairs - half
    draw = {"imul": (3 + 15 * Q) / G, "alu": (2 + 17 * Q + 2 * pairs) / G,
            "fp32": fp32_draw / G, "mufu": (4 * pairs - half) / G}
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
    elif target == "pursuit_min":
        A = n // 3
        samp["fp32"] += 2 + 6 * (A - 1)
        samp["alu"] += A - 1
        samp["mufu"] += 1
    elif target == "disk":
        samp["fp32"] += 4
        samp["mufu"] += 1
    elif target == "rel_disk6":
        samp["fp32"] += 6                   # 2 × (z diff + FFMA), FMUL + FFMA for the norm²
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

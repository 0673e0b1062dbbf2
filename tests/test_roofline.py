"""The ALU roofline model (paper_2605_18566_b200/roofline.py): hand-derived
per-eval operation counts, the draw layout of the sampler contract (R19) and the binding pipe,
checked against numbers worked out by hand here (not by calling the formula twice)."""
import pytest

from paper_2605_18566_b200 import roofline as RL


@pytest.mark.parametrize("n,G,Q", [(1, 4, 1), (2, 2, 1), (3, 4, 3), (4, 1, 1), (6, 2, 3),
                                   (8, 1, 2), (15, 1, 4), (45, 1, 12)])
def test_draw_layout(n, G, Q):
    """G = 4/gcd(n, 4) draws share ceil(G·n/4) Philox blocks when G·n ≤ 16, else one draw owns
    ceil(n/4) blocks; no normal is wasted for n = 2, 3, 6."""
    assert RL.draw_layout(n) == (G, Q)


def test_c2_counts_by_hand():
    """n = 3 disk (C2): a group of 4 draws uses 3 Philox blocks → (3 + 15·3)/4 = 12 multiplies,
    (2 + 17·3 + 2·6)/4 = 16.25 ALU (XORs + 2 mantissa builds per pair, 6 pairs). Box–Muller FP32
    in σ-scaled coordinates: one u per pair (6) and one w·r̂ per (sample, pair) — the 12 normals
    0-1-2 | 3-4-5 | 6-7-8 | 9-10-11 split the pairs (0,1)(2,3)(4,5)(6,7)(8,9)(10,11) as
    {(0,1),(2,3)}, {(2,3),(4,5)}, {(6,7),(8,9)}, {(8,9),(10,11)}: 8 — so (6 + 8)/4 = 3.5, plus the
    sample's 4 (target) + 1 (FFMA) + 1 (S) + 3 (moments) = 12.5 FP32; MUFU (4·6)/4 + SQRT + EX2
    = 8."""
    ops = RL.op_counts(3, "disk")
    assert ops["imul"] == 12.0
    assert ops["alu"] == 16.25
    assert ops["fp32"] == 12.5
    assert ops["mufu"] == 8.0
    assert ops["issue"] == 48.75


def test_c5_counts_by_hand():
    """n = 45 pair union (C5): one draw, 12 blocks → 3 + 180 = 183 multiplies; 45 normals = 22
    pairs + one cos-only → MUFU 4·23 − 1 + SQRT + EX2 = 93."""
    ops = RL.op_counts(45, "pair_union")
    assert ops["imul"] == 183
    assert ops["mufu"] == 93
    # FP32: per pair u = F − (1 − 2⁻²⁴) and w·r̂ (σ-scaled coordinates: no r̂·cos, r̂·sin), 2·23;
    # per sample 15 × (2 positions + FMUL + FFMA for |pos|²) + A·core + B + S += w + 45 moments
    assert ops["fp32"] == 2 * 23 + 15 * 4 + 1 + 1 + 45


def test_binding_pipes_with_measured_rates():
    rates = {"issue": 128.0, "fp32": 124.81, "imul": 30.37, "alu": 63.64, "mufu": 16.0}
    assert RL.roofline(3, "disk", rates=rates)["binding_pipe"] == "mufu"
    assert RL.roofline(6, "rel_disk6", rates=rates)["binding_pipe"] == "mufu"
    assert RL.roofline(15, "pair_union", rates=rates)["binding_pipe"] == "imul"
    # C2 peak: 148 SMs × 1965 MHz × 16 MUFU lane-ops/clk / 8 per eval = 5.8164e11 evals/s
    assert RL.roofline(3, "disk", rates=rates)["peak_evals_per_s"] == pytest.approx(5.8164e11)


def test_antithetic_halves_the_draw():
    a, b = RL.op_counts(3, "disk"), RL.op_counts(3, "disk", antithetic=True)
    assert b["imul"] == a["imul"] / 2
    assert b["mufu"] == pytest.approx(a["mufu"] - 0.5 * (a["mufu"] - 2))

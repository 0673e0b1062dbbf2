"""Algorithm 1's convergence test and Theorem 2's diagnostics.

CPU: the oracle's stopping-rule driver against its fixed-schedule solve (same iterates), the
residual definition, and the contraction constant / a-posteriori bound against SPEC's worked
example and geometric sequences. GPU tests live in test_gpu_parity.py."""
import math

import numpy as np
import pytest

from paper_2605_18566_b200 import inputs as I
from paper_2605_18566_b200.picard import ContractionReport, contraction_constant


def test_oracle_adaptive_equals_fixed_schedule(oracle_mod):
    O = oracle_mod
    p = I.C2.with_(N=1500, K=2)
    x = I.queries(p)[::151]
    P = O.Problem.from_preset(p, crn=False)        # fresh draws: never exactly stationary
    r = O.picard_adaptive(P, x, 0.0, 4)
    fixed = O.solve_slice(O.Problem.from_preset(p, crn=False, Kp=4), x)
    assert list(r["iters"]) == [4, 4]
    np.testing.assert_array_equal(r["v"], fixed["vhist"][:, -1])
    for j in range(2):
        prev = fixed["g0"]
        for k in range(4):
            cur = fixed["vhist"][j, k]
            eps = math.sqrt(((cur - prev) ** 2).sum() / (prev ** 2).sum())
            assert abs(r["eps"][j, k] - eps) <= 1e-12 * eps
            assert r["d_sup"][j, k] == np.abs(cur - prev).max()
            prev = cur


def test_oracle_adaptive_stops_at_first_small_residual(oracle_mod):
    O = oracle_mod
    p = I.C2.with_(N=1500, K=3)
    x = I.queries(p)[::151]
    P = O.Problem.from_preset(p, crn=False)
    full = O.picard_adaptive(P, x, 0.0, 6)
    tol = float(np.nanmedian(full["eps"]))
    r = O.picard_adaptive(P, x, tol, 6)
    for j in range(3):
        below = np.flatnonzero(full["eps"][j] < tol)
        want = (below[0] + 1) if below.size else 6
        assert r["iters"][j] == want
        np.testing.assert_array_equal(r["eps"][j, :want], full["eps"][j, :want])
        assert np.all(np.isnan(r["eps"][j, want:]))


def test_contraction_constant_spec_example():
    """G=1, c_min=1, L_D=0.01, δ=1, L_H=1, m0=1, H*=1, P*=1 → q = 0.12,
    a-posteriori factor q/(1−q) ≈ 0.1364 (Eq. contraction_const; Eq. aposteriori)."""
    q = contraction_constant(G=1, c_min=1, L_D=0.01, delta=1, L_H=1, m0=1, H_star=1, P_star=1)
    assert abs(q - 0.12) < 1e-15
    rep = ContractionReport.from_differences([1.0, 0.5], q_theory=q)
    assert rep.certified
    assert abs(rep.aposteriori[0] / 1.0 - 0.12 / 0.88) < 1e-15
    assert abs(0.12 / 0.88 - 0.1364) < 1e-4


def test_contraction_report_geometric_and_uncertified():
    d = 0.5 ** np.arange(6)
    rep = ContractionReport.from_differences(d)
    np.testing.assert_allclose(rep.q_hat, 0.5)
    assert not rep.certified and rep.aposteriori is None
    assert not ContractionReport.from_differences(d, q_theory=1.5).certified
    assert ContractionReport.from_differences([1.0]).q_hat.size == 0

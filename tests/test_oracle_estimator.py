"""Pins of the oracle's Φ pass (Cor. logsumexp P:921–931, Cor. mc_gradient P:932–941) against
closed forms, quadrature and exact per-sample-set identities — never against itself.

Statistical comparisons use the oracle's realised-weight standard errors (delta method) and
a 4.5-SE band; every such case is deterministic (fixed seeds), so the band is a fixed check.
"""
import json
import math
import os

import numpy as np
import pytest
from numpy.polynomial.hermite_e import hermegauss
from scipy import integrate, stats

HERE = os.path.dirname(os.path.abspath(__file__))
KSE = 4.5


def quad_bowl_closed_form(x, alpha0, c, sigma2):
    """g = |y|²/2 − α0, y ~ N(x, σ² I): the Gaussian integral gives
    v = |x|²/(2(1+cσ²)) − α0 + (n/(2c)) log(1+cσ²),  Dv = x/(1+cσ²)   (P:107–108 exact case)."""
    x = np.asarray(x, dtype=np.float64)
    k = c * sigma2
    return (x @ x / (2 * (1 + k)) - alpha0 + x.size / (2 * c) * math.log1p(k), x / (1 + k))


def gh_2d(f, deg=160):
    """E[f(z1, z2)], z ~ N(0, I2), by a Gauss–Hermite tensor rule."""
    t, w = hermegauss(deg)
    w = w / math.sqrt(2 * math.pi)
    Z1, Z2 = np.meshgrid(t, t, indexing="ij")
    W = np.outer(w, w)
    return float(np.sum(W * f(Z1, Z2)))


def test_golden_c1_closed_form():
    """The closed form reproduces the config-1 values stored in tests/golden (SURVEY §8(c),
    computed from P:107–108 with α0 = 0.25, n = 2, τ = 0.5, δ = 0.05)."""
    with open(os.path.join(HERE, "golden", "c1_closed_form.json")) as fh:
        gold = json.load(fh)
    for conv in ("paper", "full"):
        d = gold[conv]
        for key, x in (("v_origin", (0.0, 0.0)), ("v_11", (1.0, 1.0))):
            v, dv = quad_bowl_closed_form(x, 0.25, d["c"], d["sigma2"])
            assert abs(v - d[key]) < 5e-7
            np.testing.assert_allclose(dv, np.asarray(x) / 1.5, atol=1e-15)


@pytest.mark.parametrize("visc", ["paper", "full"])
def test_quadratic_closed_form(oracle_mod, visc):
    O = oracle_mod
    P = O.Problem(n=2, delta=0.05, T=0.5, N=1 << 16, visc=visc, target="quad_bowl",
                  tgt_params=(0.25,))
    c = 1.0 / P.delta_eff
    for qid, x in enumerate([(0.0, 0.0), (0.5, -0.25), (1.0, 1.0), (-0.9, 0.3)]):
        v, dv, diag, se = O.phi(P, x, c, P.T, qid=qid)
        vx, dvx = quad_bowl_closed_form(x, 0.25, c, P.delta_eff * P.T)
        assert abs(v - vx) < KSE * diag[3] + 1e-12
        assert np.all(np.abs(dv - dvx) < KSE * se + 1e-12)


def test_quadratic_closed_form_n45(oracle_mod):
    """Separable high-n pin: same closed form at n = 45 (small |x|, small cσ²)."""
    O = oracle_mod
    P = O.Problem(n=45, delta=0.01, T=1.0, N=1 << 14, target="quad_bowl", tgt_params=(0.25,))
    c = 10.0
    x = np.full(45, 0.05)
    v, dv, diag, se = O.phi(P, x, c, 0.5)
    vx, dvx = quad_bowl_closed_form(x, 0.25, c, 0.01 * 0.5)
    assert abs(v - vx) < KSE * diag[3]
    assert np.all(np.abs(dv - dvx) < KSE * se)


def test_constant_target_exact(oracle_mod):
    O = oracle_mod
    for N in (1, 7, 1000):
        P = O.Problem(n=3, N=N, target="const", tgt_params=(-1.75,))
        for c in (0.05, 1.0, 20.0):
            v, dv, diag, se = O.phi(P, (1.0, 2.0, 3.0), c, 0.3)
            assert abs(v - (-1.75)) < 1e-12


def test_linear_target_tilt(oracle_mod):
    """g = a·y + b: v = a·x + b − cσ²|a|²/2 and Dv = a exactly in expectation (Gaussian tilt)."""
    O = oracle_mod
    a = np.array([0.7, -1.2, 0.4])
    P = O.Problem(n=3, N=1 << 15, target="linear", tgt_params=tuple(a) + (0.3,))
    for c, tau in ((1.0, 0.5), (5.0, 0.1)):
        x = np.array([0.2, -0.4, 1.1])
        v, dv, diag, se = O.phi(P, x, c, tau)
        s2 = P.delta_eff * tau
        assert abs(v - (a @ x + 0.3 - c * s2 * a @ a / 2)) < KSE * diag[3]
        assert np.all(np.abs(dv - a) < KSE * se)


def test_disk_gauss_hermite(oracle_mod):
    """DISK target in n = 2 and the Dubins n = 3 layout: 2-D Gauss–Hermite quadrature of
    E[e^{−cg}] and E[z e^{−cg}] (z3 does not enter g, so its moment is 0 in expectation)."""
    O = oracle_mod
    c, tau, r = 2.0, 9.0, 5.0
    for n in (2, 3):
        P = O.Problem(n=n, delta=0.01, N=1 << 16, target="disk", tgt_params=(r,))
        s = math.sqrt(0.01 * tau)
        for x in ((4.8, 0.5), (-2.0, 6.0)):
            xx = np.array(list(x) + [0.3] * (n - 2))
            W = lambda z1, z2: np.exp(-c * (np.hypot(x[0] + s * z1, x[1] + s * z2) - r))
            Ew = gh_2d(W)
            v_q = -math.log(Ew) / c
            dv_q = [-(gh_2d(lambda a, b: a * W(a, b)) / Ew) / (c * s),
                    -(gh_2d(lambda a, b: b * W(a, b)) / Ew) / (c * s)] + [0.0] * (n - 2)
            v, dv, diag, se = O.phi(P, xx, c, tau, qid=7)
            assert abs(v - v_q) < KSE * diag[3]
            assert np.all(np.abs(dv - np.array(dv_q)) < KSE * se)


def test_rel_disk6_quadrature(oracle_mod):
    """REL_DISK6 depends on (y0−y3, y1−y4) ~ N(Δ, 2σ² I2); E[w z0] = E[w ζx]/√2 = −E[w z3]."""
    O = oracle_mod
    c, tau, r = 1.5, 4.0, 1.5
    P = O.Problem(n=6, delta=0.01, N=1 << 16, system="rocket6", target="rel_disk6", tgt_params=(r,))
    s = math.sqrt(0.01 * tau)
    x = np.array([1.2, 0.9, 0.1, -0.3, 0.2, -0.2])
    dx, dz = x[0] - x[3], x[1] - x[4]
    W = lambda a, b: np.exp(-c * (np.hypot(dx + math.sqrt(2) * s * a, dz + math.sqrt(2) * s * b) - r))
    Ew = gh_2d(W)
    v_q = -math.log(Ew) / c
    ex = gh_2d(lambda a, b: a * W(a, b)) / Ew / math.sqrt(2)
    ez = gh_2d(lambda a, b: b * W(a, b)) / Ew / math.sqrt(2)
    dv_q = -np.array([ex, ez, 0.0, -ex, -ez, 0.0]) / (c * s)
    v, dv, diag, se = O.phi(P, x, c, tau, qid=3)
    assert abs(v - v_q) < KSE * diag[3]
    assert np.all(np.abs(dv - dv_q) < KSE * se)


def _pair_union_quadrature_v(pos, r, sigma, c):
    """P(g > s) = Π_q P(‖pos_q + σ z_q‖ > s + r) (independent pairs; Rice / noncentral χ²₂);
    E[e^{−cg}] = e^{cr} − c ∫_{−r}^∞ e^{−cs} P(g > s) ds."""
    lam = [(np.hypot(*p) / sigma) ** 2 for p in pos]

    def surv(s):
        return float(np.prod([stats.ncx2.sf(((s + r) / sigma) ** 2, 2, l) for l in lam]))

    dist = [np.hypot(*p) for p in pos]
    lo, hi = -r, min(dist) - r + 12 * sigma
    val, _ = integrate.quad(lambda s: math.exp(-c * s) * surv(s), lo, hi, limit=400,
                            epsabs=1e-13, epsrel=1e-11)
    Ew = math.exp(c * r) - c * val
    return -math.log(Ew) / c


def test_pair_union_noncentral_chi2(oracle_mod):
    O = oracle_mod
    K, r, c, tau = 5, 1.0, 5.0, 9.0
    P = O.Problem(n=3 * K, delta=0.01, N=1 << 17, system="dubins_pairs", target="pair_union",
                  tgt_params=(r,))
    s = math.sqrt(0.01 * tau)
    x = np.zeros(3 * K)
    x[0:2] = (1.1, 0.4)
    x[3:5] = (0.9, -0.8)
    for q in range(2, K):
        x[3 * q] = 10.0 + 2.0 * q
    pos = [tuple(x[3 * q:3 * q + 2]) for q in range(K)]
    v_q = _pair_union_quadrature_v(pos, r, s, c)
    v, dv, diag, se = O.phi(P, x, c, tau, qid=1)
    assert abs(v - v_q) < KSE * diag[3]
    # gradient: central differences of the smooth quadrature value in the pair-0 coordinates
    h = 1e-4
    for d in (0, 1, 3, 4):
        xp, xm = x.copy(), x.copy()
        xp[d] += h
        xm[d] -= h
        posp = [tuple(xp[3 * q:3 * q + 2]) for q in range(K)]
        posm = [tuple(xm[3 * q:3 * q + 2]) for q in range(K)]
        g_fd = (_pair_union_quadrature_v(posp, r, s, c) - _pair_union_quadrature_v(posm, r, s, c)) / (2 * h)
        assert abs(dv[d] - g_fd) < KSE * se[d] + 1e-5


def test_jensen_bounds_and_monotone_in_c(oracle_mod):
    """Per sample set: min_i g_i ≤ v̂ ≤ mean_i g_i, and v̂ is non-increasing in c (power means)."""
    O = oracle_mod
    P = O.Problem(n=3, delta=0.01, N=4000, system="dubins_rel", target="disk", tgt_params=(5.0,))
    x = (4.0, 2.5, 1.0)
    prev = math.inf
    for c in (0.05, 0.3, 1.0, 4.0, 20.0, 200.0):
        v, dv, diag, se = O.phi(P, x, c, 1.0, qid=4)
        assert diag[0] - 1e-12 <= v <= diag[1] + 1e-12
        assert v <= prev + 1e-12
        prev = v
    # limits: c → 0 gives the mean of g, c → ∞ the min of g
    v0, _, d0, _ = O.phi(P, x, 1e-7, 1.0, qid=4)
    assert abs(v0 - d0[1]) < 1e-6
    vinf, _, dinf, _ = O.phi(P, x, 1e6, 1.0, qid=4)
    assert abs(vinf - dinf[0]) < 1e-4


def test_shift_equivariance(oracle_mod):
    """g → g + k shifts v̂ by k and leaves Dv̂ unchanged, exactly for the same samples."""
    O = oracle_mod
    P1 = O.Problem(n=2, N=3000, target="quad_bowl", tgt_params=(0.25,))
    P2 = O.Problem(n=2, N=3000, target="quad_bowl", tgt_params=(0.25 - 1.5,))
    x = (0.4, -0.3)
    v1, dv1, _, _ = O.phi(P1, x, 7.0, 0.5)
    v2, dv2, _, _ = O.phi(P2, x, 7.0, 0.5)
    assert abs((v2 - v1) - 1.5) < 1e-12
    np.testing.assert_allclose(dv2, dv1, rtol=1e-11, atol=1e-13)


def test_translation_identity(oracle_mod):
    """R4 drift hook: v_b(x) = v_0(x + bτ) for identical z."""
    O = oracle_mod
    P = O.Problem(n=3, delta=0.01, N=2000, system="dubins_rel", target="disk", tgt_params=(5.0,))
    x = np.array([3.0, -4.5, 0.2])
    b = np.array([1.5, 2.0, -0.7])
    tau = 0.6
    v1, dv1, _, _ = O.phi(P, x, 3.0, tau, drift=b)
    v2, dv2, _, _ = O.phi(P, x + b * tau, 3.0, tau)
    assert v1 == v2
    np.testing.assert_array_equal(dv1, dv2)


def test_tau_zero_returns_g_and_dg(oracle_mod):
    O = oracle_mod
    P = O.Problem(n=3, system="dubins_rel", target="disk", tgt_params=(5.0,))
    x = np.array([3.0, 4.0, 1.0])
    v, dv, _, _ = O.phi(P, x, 2.0, 0.0)
    assert v == 0.0
    np.testing.assert_allclose(dv, [0.6, 0.8, 0.0])


@pytest.mark.parametrize("target,n,params", [
    ("quad_bowl", 4, (0.25,)), ("disk", 3, (5.0,)), ("rel_disk6", 6, (1.5,)),
    ("pair_union", 15, (1.0,)), ("linear", 3, (0.5, -1.0, 2.0, 0.1))])
def test_target_gradient_matches_finite_differences(oracle_mod, target, n, params):
    O = oracle_mod
    P = O.Problem(n=n, target=target, tgt_params=params)
    rng = np.random.default_rng(3)
    for _ in range(5):
        x = rng.uniform(-3, 3, n)
        g = O.dg(P, x)
        h = 1e-6
        fd = np.array([(O.g(P, x + h * e) - O.g(P, x - h * e)) / (2 * h) for e in np.eye(n)])
        np.testing.assert_allclose(g, fd, atol=1e-7)


def test_target_values(oracle_mod):
    O = oracle_mod
    P = O.Problem(n=3, target="disk", tgt_params=(5.0,))
    assert O.g(P, (3.0, 4.0, 9.0)) == 0.0               # on the capture circle
    P = O.Problem(n=6, target="rel_disk6", tgt_params=(1.5,))
    assert abs(O.g(P, (1.0, 2.0, 0.0, 1.0, 0.5, 0.0)) - 0.0) < 1e-15
    P = O.Problem(n=9, target="pair_union", tgt_params=(1.0,))
    assert O.g(P, (10, 0, 0, 3, 4, 0, 0, -8, 0)) == 4.0   # nearest pair at distance 5
    assert list(O.dg(P, (0, 0, 0, 3, 4, 0, 9, 9, 0))) == [1, 0, 0, 0, 0, 0, 0, 0, 0]  # e1 at ρ = 0
    P = O.Problem(n=2, target="quad_bowl", tgt_params=(0.25,))
    assert O.g(P, (1.0, 1.0)) == 0.75


# ---- Laplace-tilted proposal (R28) -----------------------------------------------
def test_tilted_linear_target_is_zero_variance(oracle_mod):
    """g = a·y + b: μ = x − cσ²a is the exact mode, the likelihood-ratio weights are constant and
    v̂ equals the Gaussian-tilt value a·x + b − cσ²|a|²/2 for ANY N (even N = 1)."""
    O = oracle_mod
    a = np.array([0.7, -1.2, 0.4])
    for N in (1, 17, 3000):
        P = O.Problem(n=3, N=N, target="linear", tgt_params=tuple(a) + (0.3,), proposal="laplace")
        for c, tau in ((1.0, 0.5), (5.0, 0.1)):
            x = np.array([0.2, -0.4, 1.1])
            v, dv, diag, se = O.phi(P, x, c, tau)
            s2 = P.delta_eff * tau
            assert abs(v - (a @ x + 0.3 - c * s2 * a @ a / 2)) < 1e-12
            assert abs(diag[2] - N) < 1e-6 * N           # ESS = N: every weight equal


def test_tilted_quadratic_closed_form_and_ess(oracle_mod):
    """Quadratic bowl: the tilted estimator matches the closed form within its SE
    and, where the plain weights collapse (c|x|² large), has a far larger effective sample size."""
    O = oracle_mod
    c = 20.0
    for x in ((0.0, 0.0), (1.0, 1.0), (-0.9, 0.3)):
        Pp = O.Problem(n=2, delta=0.05, T=0.5, N=1 << 15, target="quad_bowl", tgt_params=(0.25,))
        Pt = O.Problem(n=2, delta=0.05, T=0.5, N=1 << 15, target="quad_bowl", tgt_params=(0.25,),
                       proposal="laplace")
        vx, dvx = quad_bowl_closed_form(x, 0.25, c, 0.05 * 0.5)
        vt, dvt, dt, st = O.phi(Pt, x, c, 0.5, qid=3)
        vp, dvp, dp, sp = O.phi(Pp, x, c, 0.5, qid=3)
        assert abs(vt - vx) < KSE * dt[3] + 1e-12
        assert np.all(np.abs(dvt - dvx) < KSE * st + 1e-12)
        if np.dot(x, x) > 1:
            assert dt[2] > 3 * dp[2]                     # ESS
            assert dt[3] < dp[3] / 2                     # SE of v


def test_tilted_agrees_with_plain_on_games(oracle_mod):
    """Disk (Dubins) and pair-union targets: tilted and plain estimates of the same Φ agree
    within their combined standard errors (both estimate E_p[e^{−cg}])."""
    O = oracle_mod
    cases = [(3, "dubins_rel", "disk", (5.0,), (4.0, 3.5, 1.0), 20.0, 1.0),
             (15, "dubins_pairs", "pair_union", (1.0,), tuple([1.1, 0.4, 0.0, 0.9, -0.8, 0.0] + [12.0, 0, 0] * 3), 5.0, 0.5)]
    for n, system, target, tp, x, c, tau in cases:
        kw = dict(n=n, delta=0.01, N=1 << 15, system=system, target=target, tgt_params=tp)
        vp, dvp, dp, sp = O.phi(O.Problem(**kw), x, c, tau, qid=5)
        vt, dvt, dt, st = O.phi(O.Problem(**kw, proposal="laplace"), x, c, tau, qid=5)
        assert abs(vp - vt) < KSE * math.hypot(dp[3], dt[3])
        assert np.all(np.abs(dvp - dvt) < KSE * np.hypot(sp, st) + 1e-9)


# ---- the oracle's statistical yardstick ---------------------------------
@pytest.mark.parametrize("case", ["bowl", "disk", "pair_union"])
def test_standard_errors_match_seed_spread(oracle_mod, case):
    """Pin of orc_phi's delta-method standard errors — diag[3] for v̂ and se_dv for each Dv̂
    component — which set the width of every MC-vs-quadrature pin above. Thm 1
    makes v̂ a sample-mean functional with O(N^-½) spread; over R = 2048 independent seeds at a
    fixed (x, c, τ) the empirical standard deviation of v̂ and of every Dv̂ component must match
    the mean of the per-run SE estimates within ±10 %: the χ² 99.9 % band of a 2048-sample
    standard deviation is ±5.1 %, the rest covers the O(1/N) delta-method bias. A dropped 1/c,
    1/σ or √N, or S in place of S², misses by a factor ≥ √2."""
    O = oracle_mod
    if case == "bowl":
        kw = dict(n=2, delta=0.05, visc="paper", system="quadratic", target="quad_bowl",
                  tgt_params=(0.25,))
        x, c, tau = np.array([0.3, -0.2]), 20.0, 0.2
    elif case == "disk":
        kw = dict(n=2, delta=0.01, system="quadratic", target="disk", tgt_params=(1.0,))
        x, c, tau = np.array([1.1, 0.4]), 6.0, 1.0
    else:
        kw = dict(n=15, delta=0.02, system="dubins_pairs", target="pair_union", tgt_params=(1.0,))
        x = np.zeros(15)
        x[0], x[1], x[3], x[4] = 1.3, 0.2, 0.9, -1.2
        x[6:] = np.tile([4.0, 0.0, 0.0], 3)
        c, tau = 3.0, 1.0
    R, N = 2048, 4096
    v = np.zeros(R)
    dv = np.zeros((R, x.size))
    se_v = np.zeros(R)
    se_dv = np.zeros((R, x.size))
    for r in range(R):
        P = O.Problem(N=N, seed=0xC0FFEE00 + 7919 * r, **kw)
        v[r], dv[r], diag, se_dv[r] = O.phi(P, x, c, tau, qid=r, jw=1, kw=0)
        se_v[r] = diag[3]
    lo, hi = stats.chi2.ppf([5e-4, 1 - 5e-4], R - 1) / (R - 1)
    assert 0.94 < math.sqrt(lo) and math.sqrt(hi) < 1.06          # the ±5.1 % band, R = 2048
    ratio_v = v.std(ddof=1) / se_v.mean()
    ratio_dv = dv.std(axis=0, ddof=1) / se_dv.mean(axis=0)
    print(f"{case}: std/SE v {ratio_v:.4f}, Dv {np.round(ratio_dv, 4)}")
    assert abs(ratio_v - 1.0) < 0.10, ratio_v
    assert np.all(np.abs(ratio_dv - 1.0) < 0.10), ratio_dv

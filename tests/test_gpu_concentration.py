"""GPU concentration harness: the CUDA estimator over tens of
thousands of independent Philox streams (distinct global query ids at one state), checked
against mathematics — not against the oracle:

* mean of v̂ = closed form + the delta-method bias (1/(2c))·CV²/N, within 4 SE;
* spread of v̂ = the delta-method SE CV/(c√N), and its log-log slope in N is −1/2 (Thm 1's
  O(N^{-1/2}));
* mean of Dv̂ = x/(1+k) + (ρ/N)·x·(1/(1+k) − 2/(1+2k)), k = cσ², ρ = E[w²]/E[w]²: the
  O(1/N) bias of the self-normalised (ratio) gradient estimator, from the delta method with
  the bowl's Gaussian moments E[w z] ∝ −cσx/(1+k), E[w² z] ∝ −2cσx/(1+2k);
* Thm 1's Hoeffding tail bound and Cor. 1's sample size (P:273–282, S:222 scenario)
  hold empirically; the sampler's support (|z_d| ≤ sqrt(48 ln 2)) bounds g as Thm 1 assumes.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

R = 32768
ZMAX = math.sqrt(48 * math.log(2))


def draws(N, x, c, tau, target="quad_bowl", tgt=(0.25,), delta=0.05, n=2):
    s = Solver(SolverConfig(n=n, delta=delta, N=N, seed=0xC0FFEE, system="quadratic",
                            target=target, tgt_params=tgt))
    xs = np.tile(np.asarray(x, np.float32), (R, 1))
    v, dv = s.value_grad(xs, np.full(R, c, np.float32), tau, j_tag=9, k_tag=0)
    return v.cpu().numpy().astype(np.float64), dv.cpu().numpy().astype(np.float64)


def bowl_truth(x, c, s2, n=2, a0=0.25):
    x = np.asarray(x, np.float64)
    k = c * s2
    v = x @ x / (2 * (1 + k)) - a0 + n / (2 * c) * math.log1p(k)
    cv2 = ((1 + k) ** 2 / (1 + 2 * k)) ** (n / 2) * math.exp(c * (x @ x) * (1 / (1 + k) - 1 / (1 + 2 * k))) - 1
    return v, x / (1 + k), cv2


def test_mean_bias_and_spread_match_theory():
    x, c, tau, delta = (0.3, -0.2), 20.0, 0.5, 0.05
    s2 = delta * tau
    v_true, dv_true, cv2 = bowl_truth(x, c, s2)
    for N in (256, 1024):
        v, dv = draws(N, x, c, tau)
        se = math.sqrt(cv2 / N) / c                    # delta-method SE of v̂
        bias = cv2 / (2 * c * N)                       # E[v̂] − v to O(1/N)
        assert abs(v.mean() - (v_true + bias)) < 4 * se / math.sqrt(R) + 2e-6
        assert abs(v.std(ddof=1) / se - 1) < 0.05
        sd_dv = dv.std(axis=0, ddof=1)
        k = c * s2
        dv_bias = (1 + cv2) / N * np.asarray(x) * (1 / (1 + k) - 2 / (1 + 2 * k))
        assert np.all(np.abs(dv.mean(axis=0) - (dv_true + dv_bias)) < 4 * sd_dv / math.sqrt(R) + 1e-5)


def test_concentration_rate_slope():
    x, c, tau = (0.3, -0.2), 20.0, 0.5
    Ns = [64, 256, 1024, 4096]
    sds = [draws(N, x, c, tau)[0].std(ddof=1) for N in Ns]
    slope = np.polyfit(np.log(Ns), np.log(sds), 1)[0]
    assert abs(slope + 0.5) < 0.03


def test_theorem1_hoeffding_tail():
    """P(|v̂ − v| ≥ ε) ≤ 2 exp(−2Nμ²(1 − e^{−cε})²/(β − α)²), α, β = e^{−c g_max}, e^{−c g_min}
    with g bounded on the sampler's support."""
    x, c, tau, delta = np.array([0.3, -0.2]), 20.0, 0.5, 0.05
    s2 = delta * tau
    v_true, _, _ = bowl_truth(x, c, s2)
    sig = math.sqrt(s2)
    ymax = np.abs(x) + sig * ZMAX
    g_max, g_min = 0.5 * float(ymax @ ymax) - 0.25, -0.25
    alpha, beta = math.exp(-c * g_max), math.exp(-c * g_min)
    mu = math.exp(-c * v_true)
    for N, eps in ((256, 0.02), (1024, 0.01)):
        v, _ = draws(N, x, c, tau)
        bound = min(1.0, 2 * math.exp(-2 * N * mu**2 * (1 - math.exp(-c * eps)) ** 2 / (beta - alpha) ** 2))
        rate = float(np.mean(np.abs(v - v_true) >= eps))
        assert rate <= bound + 3 * math.sqrt(max(bound * (1 - bound), 1e-12) / R)


def test_corollary1_sample_size_scenario():
    """S:222 / Cor. 1: c = 1, g ∈ [0, 1], ε = 0.1 ⇒ N = 276 keeps P(|v̂ − v| ≥ ε) ≤ α = e^{−1}.
    g ∈ [0, 1] on the support: disk target, x at distance r + 0.5 from the centre, σ = 0.06."""
    from numpy.polynomial.hermite_e import hermegauss

    r, c, eps, N = 5.0, 1.0, 0.1, 276
    sig = 0.06
    tau = sig**2 / 0.01
    x = (r + 0.5, 0.0)
    assert 0.5 - sig * ZMAX * math.sqrt(2) > 0 and 0.5 + sig * ZMAX * math.sqrt(2) < 1
    v, _ = draws(N, x, c, tau, target="disk", tgt=(r,), delta=0.01)
    t, w = hermegauss(120)
    w = w / math.sqrt(2 * math.pi)
    Z1, Z2 = np.meshgrid(t, t, indexing="ij")
    Ew = float(np.sum(np.outer(w, w) * np.exp(-c * (np.hypot(x[0] + sig * Z1, sig * Z2) - r))))
    v_true = -math.log(Ew) / c
    rate = float(np.mean(np.abs(v - v_true) >= eps))
    assert rate <= math.exp(-1) + 3 * math.sqrt(math.exp(-1) * (1 - math.exp(-1)) / R)
    assert abs(v.mean() - v_true) < 1e-3

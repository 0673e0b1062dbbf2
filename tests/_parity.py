"""Parity helpers shared by the GPU tests: the R20 tolerances (north_star: 2e-4 relative on v,
1e-3 on Dv), with the floors DESIGN.md §3 derives for the BRT boundary where v ≈ 0."""
import numpy as np

V_RTOL = 2e-4
DV_RTOL = 1e-3
FLOOR = 1e-2


def v_violations(v_gpu, v_ref, rtol=V_RTOL):
    v_gpu = np.asarray(v_gpu, dtype=np.float64)
    v_ref = np.asarray(v_ref, dtype=np.float64)
    floor = FLOOR * np.abs(v_ref).max()
    bound = rtol * np.maximum(np.abs(v_ref), floor)
    err = np.abs(v_gpu - v_ref)
    return err / np.maximum(bound, 1e-300)


def dv_violations(dv_gpu, dv_ref, rtol=DV_RTOL):
    dv_gpu = np.asarray(dv_gpu, dtype=np.float64)
    dv_ref = np.asarray(dv_ref, dtype=np.float64)
    nref = np.linalg.norm(dv_ref, axis=-1)
    floor = FLOOR * nref.max()
    bound = rtol * np.maximum(nref, floor)
    err = np.linalg.norm(dv_gpu - dv_ref, axis=-1)
    return err / np.maximum(bound, 1e-300)


def assert_v(v_gpu, v_ref, what="v", rtol=V_RTOL):
    r = v_violations(v_gpu, v_ref, rtol)
    worst = int(np.argmax(r))
    assert r.max() <= 1.0, (f"{what}: worst query {worst} ratio {r.max():.3g} "
                            f"gpu={np.ravel(v_gpu)[worst]!r} ref={np.ravel(v_ref)[worst]!r}")


def assert_dv(dv_gpu, dv_ref, what="dv", rtol=DV_RTOL):
    r = dv_violations(dv_gpu, dv_ref, rtol)
    worst = int(np.argmax(r))
    assert r.max() <= 1.0, (f"{what}: worst query {worst} ratio {r.max():.3g} "
                            f"gpu={np.asarray(dv_gpu)[worst]!r} ref={np.asarray(dv_ref)[worst]!r}")


# The frozen coefficient c = Γ(x, Dv) is an intermediate, not an output the north_star
# tolerances name. Γ = 2H/(δ|p|²) is ill-conditioned where H(x, p) ≈ 0 (the interior band of
# the clamp, R8): a tiny relative change of Dv moves c a lot. Its parity bound is therefore the
# first-order perturbation bound  |Δc| ≤ 2e-4·max(|c|, floor) + ‖∇_pΓ(x, p)‖·ε·max(‖p‖, m0)
# with p the oracle's own Dv of the previous iterate (Dg(x) for c^(0)) and ε = 1e-4, ten times
# tighter than the Dv tolerance.
C_DV_EPS = 1e-4


def c_violations(O, P, x, c_gpu, c_ref, p_ref):
    """Ratios |Δc| / bound for one iterate; x[M][n], p_ref[M][n] (oracle Dv or Dg)."""
    c_gpu = np.asarray(c_gpu, dtype=np.float64)
    c_ref = np.asarray(c_ref, dtype=np.float64)
    floor = FLOOR * np.abs(c_ref).max()
    out = np.zeros(len(c_ref))
    for m in range(len(c_ref)):
        err = abs(c_gpu[m] - c_ref[m])
        base = V_RTOL * max(abs(c_ref[m]), floor)
        if err <= base:
            continue
        xm = np.asarray(x[m], dtype=np.float64)
        sens = O.gamma_sensitivity(P, xm, p_ref[m])
        out[m] = err / (base + sens * C_DV_EPS * max(np.linalg.norm(p_ref[m]), P.m0))
    return out


def assert_c_history(O, P, x, chist_gpu, ref):
    """Check every frozen coefficient c^(k) of every horizon against the perturbation bound."""
    x = np.asarray(x, dtype=np.float64)
    dg = np.stack([O.dg(P, xm) for xm in x])
    for j in range(P.K):
        for k in range(P.Kp):
            p_ref = dg if k == 0 else ref["dvhist"][j, k - 1]
            r = c_violations(O, P, x, chist_gpu[j, k], ref["chist"][j, k], p_ref)
            worst = int(np.argmax(r))
            assert r.max() <= 1.0, (f"chist[{j},{k}] worst query {worst} ratio {r.max():.3g} "
                                    f"gpu={chist_gpu[j, k][worst]!r} ref={ref['chist'][j, k][worst]!r}")

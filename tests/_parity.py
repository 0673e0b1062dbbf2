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


# Picard iterates in the non-contractive regime. Theorem 2 guarantees contraction
# only when q < 1; where H(x, Dv) ≈ 0 and c is unclamped (R8) the map c ↦ Γ(x, Dv(Φ(c))) can be
# expansive, and ANY rounding difference between two implementations grows geometrically with
# k. There the allowed deviation at iterate k is the first-order propagation, along the
# oracle's own trajectory, of a relative Dv perturbation ε = 1e-4 per iterate:
#   Δc⁽⁰⁾ = ‖∇_pΓ(x, Dg)‖·ε‖Dg‖,
#   Δv⁽ᵏ⁾ = 2e-4·max(|v|, floor) + |∂v/∂c|·Δc⁽ᵏ⁾,   ΔDv⁽ᵏ⁾ = ε‖Dv‖ + ‖∂Dv/∂c‖·Δc⁽ᵏ⁾,
#   Δc⁽ᵏ⁺¹⁾ = 2e-4·|c⁽ᵏ⁺¹⁾| + ‖∇_pΓ(x, Dv⁽ᵏ⁾)‖·ΔDv⁽ᵏ⁾,
# with ∂Φ/∂c from central differences of the oracle's Φ at its own c (oracle-only data).
# Contractive queries never reach this path: their plain R20 check passes.
def propagated_bounds(O, P, x, qid, j, c_ref, v_ref, dv_ref, floor):
    """Allowed |Δv|, |Δc| and ‖ΔDv‖ per iterate k for one query and horizon j (1-based)."""
    x = np.asarray(x, dtype=np.float64)
    tau = j * P.T / P.K
    p0 = O.dg(P, x)
    dc = O.gamma_sensitivity(P, x, p0) * C_DV_EPS * max(np.linalg.norm(p0), P.m0)
    bv, bc, bd = np.zeros(P.Kp), np.zeros(P.Kp), np.zeros(P.Kp)
    for k in range(P.Kp):
        c = float(c_ref[k])
        bc[k] = V_RTOL * abs(c) + dc
        h = 1e-4 * c
        kw = 0 if P.crn else k
        vp, dvp, _, _ = O.phi(P, x, c + h, tau, qid=int(qid), jw=j, kw=kw)
        vm, dvm, _, _ = O.phi(P, x, c - h, tau, qid=int(qid), jw=j, kw=kw)
        dv_dc = abs(vp - vm) / (2 * h)
        ddv_dc = np.linalg.norm(dvp - dvm) / (2 * h)
        bv[k] = V_RTOL * max(abs(float(v_ref[k])), floor) + dv_dc * dc
        bdv = C_DV_EPS * np.linalg.norm(dv_ref[k]) + ddv_dc * dc
        bd[k] = max(bdv, DV_RTOL * np.linalg.norm(dv_ref[k]))
        if k + 1 < P.Kp:
            dc = V_RTOL * abs(float(c_ref[k + 1])) + O.gamma_sensitivity(P, x, dv_ref[k]) * bdv
    return bv, bc, bd


# R27 allowance, capped at the rates measured on the complete C2 slice (round 1: 1 of 102,010
# (query, horizon) units and 2 of 10,201 final outputs needed the propagated bound): at most
# 0.1 % of units and 0.05 % of final outputs — at least one, for the small sampled sets that
# deliberately include the interior-c band (R8) where Γ is expansive.
R27_UNIT_FRAC = 1e-3
R27_OUTPUT_FRAC = 5e-4


def r27_cap(count, frac):
    return max(1, int(frac * count))


def assert_picard_history(O, P, x, qids, vhist_gpu, chist_gpu, ref, what=""):
    """vhist and chist at every (j, k): the plain R20 / R25 checks, and for a (query, horizon)
    that fails them, the propagated non-contractive bound above. Returns the number of
    (query, horizon) pairs that needed the propagated bound, which must stay within the R27 cap
    (printed, with the ids)."""
    x = np.asarray(x, dtype=np.float64)
    M = x.shape[0]
    floor = FLOOR * np.abs(ref["vhist"]).max()
    dg = np.stack([O.dg(P, xm) for xm in x])
    # vectorised pre-check: units whose every iterate passes plain R20 on v and c's base term
    # need no per-iterate work (c_violations' first test is exactly the base term)
    vr, cr = np.asarray(ref["vhist"]), np.asarray(ref["chist"])
    vg = np.asarray(vhist_gpu, dtype=np.float64)
    cg = np.asarray(chist_gpu, dtype=np.float64)
    quick = ((np.abs(vg - vr) <= V_RTOL * np.maximum(np.abs(vr), floor))
             & (np.abs(cg - cr) <= V_RTOL * np.abs(cr))).all(axis=1)        # [K][M]
    needed = 0
    for m in range(M):
        for j in range(P.K):
            if quick[j, m]:
                continue
            base_ok = True
            for k in range(P.Kp):
                vr = ref["vhist"][j, k, m]
                if abs(vhist_gpu[j, k, m] - vr) > V_RTOL * max(abs(vr), floor):
                    base_ok = False
                    break
                p_ref = dg[m] if k == 0 else ref["dvhist"][j, k - 1, m]
                if c_violations(O, P, x[m:m + 1], [chist_gpu[j, k, m]], [ref["chist"][j, k, m]],
                                p_ref[None])[0] > 1.0:
                    base_ok = False
                    break
            if base_ok:
                continue
            needed += 1
            print(f"R27 {what}: query {int(qids[m])} horizon {j + 1} judged by the propagated bound")
            bv, bc, _ = propagated_bounds(O, P, x[m], qids[m], j + 1, ref["chist"][j, :, m],
                                       ref["vhist"][j, :, m], ref["dvhist"][j, :, m], floor)
            for k in range(P.Kp):
                dv = abs(vhist_gpu[j, k, m] - ref["vhist"][j, k, m])
                dc = abs(chist_gpu[j, k, m] - ref["chist"][j, k, m])
                assert dv <= bv[k] and dc <= bc[k], (
                    f"query {qids[m]} horizon {j} iterate {k}: |Δv| {dv:.3g} (bound {bv[k]:.3g}), "
                    f"|Δc| {dc:.3g} (bound {bc[k]:.3g})")
    units = M * P.K
    print(f"R27 {what}: {needed} of {units} (query, horizon) units needed the propagated bound "
          f"(cap {r27_cap(units, R27_UNIT_FRAC)})")
    assert needed <= r27_cap(units, R27_UNIT_FRAC), f"{needed} units needed the R27 band"
    return needed


def _final_outputs_within(O, P, x, qids, g, ref, sel=None):
    """v, Dv and tube at τ_K: R20, except for queries whose last horizon is non-contractive,
    which are covered by assert_picard_history's propagated bound on vhist[K−1][Kp−1] (= v)."""
    take = (lambda a: a[sel]) if sel is not None else (lambda a: a)
    vg, dvg, tg = take(g["v"]), take(g["dv"]), take(g["tube"])
    okv = v_violations(vg, ref["v"]) <= 1.0
    okd = dv_violations(dvg, ref["dv"]) <= 1.0
    okt = v_violations(tg, ref["tube"]) <= 1.0
    bad = np.flatnonzero(~(okv & okd & okt))
    floor = 1e-2 * np.abs(ref["vhist"]).max()
    for m in bad:                                   # must be explained by the propagated bound
        bv, _, bd = propagated_bounds(O, P, x[m], qids[m], P.K, ref["chist"][-1, :, m],
                                      ref["vhist"][-1, :, m], ref["dvhist"][-1, :, m], floor)
        assert abs(vg[m] - ref["v"][m]) <= bv[-1], f"v at query {qids[m]}"
        assert np.linalg.norm(dvg[m] - ref["dv"][m]) <= bd[-1], f"Dv at query {qids[m]}"
        assert abs(tg[m] - ref["tube"][m]) <= max(bv[-1], 2e-4 * max(abs(ref["tube"][m]), floor))
    print(f"R27: {len(bad)} of {len(vg)} final outputs judged by the propagated bound "
          f"(ids {[int(qids[m]) for m in bad]}; cap {r27_cap(len(vg), R27_OUTPUT_FRAC)})")
    assert len(bad) <= r27_cap(len(vg), R27_OUTPUT_FRAC), f"{len(bad)} queries outside R20 at τ_K"


# Teacher forcing: Φ alone at the oracle's OWN coefficient history. Under
# common random numbers a pass is a function of (query, horizon, c), so every iterate (j, k) of a
# trajectory maps to one item (m, j, float32(chist[j, k, m])); both sides evaluate Φ there with
# τ_j as the fp32 value hjmc_value_grad receives and counter tags (j + 1, 0).
def teacher_items(chist):
    """Unique (m, j, float32 c) items of chist[K][Kp][M] and, per (j, k, m), the item index."""
    K, Kp, M = chist.shape
    cf = np.asarray(chist).astype(np.float32)
    keys = {}
    index = np.zeros((K, Kp, M), dtype=np.int64)
    for j in range(K):
        for k in range(Kp):
            for m, c in enumerate(cf[j, k].tolist()):
                index[j, k, m] = keys.setdefault((m, j, c), len(keys))
    items = sorted(keys, key=keys.get)
    m = np.array([t[0] for t in items], dtype=np.int64)
    j = np.array([t[1] for t in items], dtype=np.int64)
    c = np.array([t[2] for t in items], dtype=np.float32)
    return m, j, c, index


def teacher_tau(T, K, j0):
    """τ_j (j0 = 0-based horizon) as the fp32 value hjmc_value_grad receives."""
    return np.float32((j0 + 1) * T / K)

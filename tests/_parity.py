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

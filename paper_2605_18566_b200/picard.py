"""Algorithm 1 with its convergence test, driven through the C-ABI's stepwise Picard calls,
plus Theorem 2's contraction diagnostics.

Algorithm 1 stops when ε = ‖v^(k+1) − v^(k)‖/‖v^(k)‖ < tol (step 5; relative L2
over the slice's queries, R11), per horizon j. The norms are slice-wide — with queries sharded
over GPUs the per-rank partial sums (hjmc_picard_pass) are all-reduced before the decision, so
every rank takes the same decision. Every Φ pass and Γ update runs in the CUDA kernels; this
module only marshals: the shards' residual partials are combined by one all-reduce (plumbing),
and the stopping test (hjmc_picard_decide) and the tube with its BRAT clamp (hjmc_tube) run in
the library.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


def contraction_constant(G: float, c_min: float, L_D: float, delta: float, L_H: float,
                         m0: float, H_star: float, P_star: float) -> float:
    """q of Assumption 1 item 5 (Eq. contraction_const; R18 uses 2G/c_min):
    q = (2G/c_min)·(2 L_D/δ)·(L_H/m0² + 2 H* P*/m0⁴) — hjmc_contraction_constant."""
    return float(_lib.load().hjmc_contraction_constant(G, c_min, L_D, delta, L_H, m0, H_star,
                                                        P_star))


@dataclass
class ContractionReport:
    """Theorem 2 diagnostics from the sup-norm Picard differences d_k = ‖v^(k+1) −
    v^(k)‖∞: empirical ratios q̂_k = d_k / d_{k−1}; with a theoretical q < 1, the geometric
    bound d_k ≤ q^k d_0 (Eq. gamma-lip-cauchy) and the a-posteriori error bound
    ‖v^(k) − v*‖∞ ≤ q/(1−q)·‖v^(k) − v^(k−1)‖∞ (Eq. aposteriori-error)."""

    d_sup: np.ndarray
    q_hat: np.ndarray
    q_theory: float | None
    aposteriori: np.ndarray | None
    certified: bool

    @classmethod
    def from_differences(cls, d_sup, q_theory: float | None = None) -> "ContractionReport":
        """Marshals d_sup through hjmc_contraction_report (ratios and the a-posteriori bound
        are computed in the library)."""
        d = np.ascontiguousarray(d_sup, dtype=np.float64)
        q_hat = np.zeros(max(d.size - 1, 0))
        apost = np.zeros(d.size)
        q = float(q_theory) if q_theory is not None else -1.0
        rc = _lib.load().hjmc_contraction_report(
            d.ctypes.data_as(C.c_void_p), d.size, q, q_hat.ctypes.data_as(C.c_void_p),
            apost.ctypes.data_as(C.c_void_p))
        if rc < 0:
            raise _lib.HjmcError(1, "contraction_report")
        certified = rc == 1
        return cls(d, q_hat, q_theory, apost if certified else None, certified)


def solve_adaptive(solver, x, tol: float, max_iter: int, qid_base: int = 0, qid=None,
                   drift=None, allreduce=None, want_dv: bool = True, log=None):
    """Run Algorithm 1 per horizon until ε_j(k) < tol or max_iter passes.

    allreduce(partials[K][3] float64) -> partials: combine shards (sum cols 0–1, max col 2);
    None for a single process. log: optional callable receiving one JSON-serialisable record
    per Picard iteration (k, active horizons, ε_j(k), sup-norm differences, wall ms, max|v|,
    min/max c over the active rows; the per-iteration record of S:316–317). Returns a dict:
    v, dv, c [K][M](…) device tensors of each horizon's final iterate, iters [K],
    eps [K][max_iter], d_sup [K][max_iter] (NaN past the stop), tube [M] =
    max(min(g, min_j v_j), ℓ) (hjmc_tube: running min with the BRAT clamp), converged [K]."""
    import time
    t = solver.torch
    cfg = solver.cfg
    x = solver._as_query(x)
    M, K, n = x.shape[0], cfg.K, cfg.n
    q = solver._as_dev(qid, t.int32) if qid is not None else None
    b = solver._as_dev(drift) if drift is not None else None
    L = solver.L
    stream = solver._stream()
    solver._check(L.hjmc_picard_begin(solver.h, C.c_void_p(x.data_ptr()),
                                      C.c_void_p(q.data_ptr()) if q is not None else None,
                                      qid_base, M, C.c_void_p(b.data_ptr()) if b is not None else None,
                                      stream))
    v = t.empty((K, M), device=solver.device)
    dv = t.empty((K, M, n), device=solver.device) if want_dv else None
    c = t.empty((K, M), device=solver.device)
    active = np.ones(K, dtype=np.uint8)
    iters = np.zeros(K, dtype=np.int64)
    eps = np.full((K, max_iter), np.nan)
    dsup = np.full((K, max_iter), np.nan)
    part = np.zeros((K, 3), dtype=np.float64)
    for k in range(max_iter):
        if not active.any():
            break
        t0 = time.perf_counter()
        was_active = np.flatnonzero(active)
        solver._check(L.hjmc_picard_pass(
            solver.h, k, active.ctypes.data_as(C.c_void_p), C.c_void_p(v.data_ptr()),
            C.c_void_p(dv.data_ptr()) if dv is not None else None, C.c_void_p(c.data_ptr()),
            part.ctypes.data_as(C.c_void_p), stream))
        tot = np.ascontiguousarray(allreduce(part.copy()) if allreduce is not None else part)
        iters[was_active] = k + 1
        e_k = np.empty(K)
        d_k = np.empty(K)
        left = C.c_int32()
        solver._check(L.hjmc_picard_decide(tot.ctypes.data_as(C.c_void_p), K, float(tol),
                                           active.ctypes.data_as(C.c_void_p),
                                           e_k.ctypes.data_as(C.c_void_p),
                                           d_k.ctypes.data_as(C.c_void_p), C.byref(left)))
        eps[was_active, k] = e_k[was_active]
        dsup[was_active, k] = d_k[was_active]
        if log is not None:
            rows = t.as_tensor(was_active, device=solver.device)
            va, ca = v.index_select(0, rows), c.index_select(0, rows)
            log({"k": k, "horizons": [int(j) + 1 for j in was_active],
                 "eps": [float(eps[j, k]) for j in was_active],
                 "d_sup": [float(dsup[j, k]) for j in was_active],
                 "ms": 1e3 * (time.perf_counter() - t0), "max_abs_v": float(va.abs().max()),
                 "c_min": float(ca.min()), "c_max": float(ca.max())})
    tube = t.empty(M, device=solver.device)
    solver._check(L.hjmc_tube(solver.h, C.c_void_p(x.data_ptr()), M, C.c_void_p(v.data_ptr()),
                              C.c_void_p(tube.data_ptr()), stream))
    return {"v": v, "dv": dv, "c": c, "iters": iters, "eps": eps, "d_sup": dsup, "tube": tube,
            "converged": ~active.astype(bool)}


def torch_allreduce(group=None):
    """An allreduce for solve_adaptive over torch.distributed (NCCL or gloo)."""
    import torch
    import torch.distributed as dist

    def f(part):
        s = torch.from_numpy(np.ascontiguousarray(part[:, :2]))
        m = torch.from_numpy(np.ascontiguousarray(part[:, 2]))
        if dist.get_backend(group) == "nccl":
            s, m = s.cuda(), m.cuda()
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
        out = part.copy()
        out[:, :2] = s.cpu().numpy()
        out[:, 2] = m.cpu().numpy()
        return out

    return f


def solve_adaptive_device(solver, x, tol: float, max_iter: int, qid_base: int = 0, qid=None,
                          drift=None, want_dv: bool = True):
    """Algorithm 1 with its stopping test in ONE device-resident call (hjmc_picard_solve: a CUDA
    graph whose conditional while-node loops pass → residual → decision with no host round
    trip). Single process only (sharded slices need the all-reduce of solve_adaptive). Returns
    the same dict as solve_adaptive without the log: v, dv, c [K][M](…) tensors, iters [K],
    eps / d_sup [K][max_iter] (NaN past the stop), tube [M], converged [K]."""
    t = solver.torch
    cfg = solver.cfg
    x = solver._as_query(x)
    M, K, n = x.shape[0], cfg.K, cfg.n
    q = solver._as_dev(qid, t.int32) if qid is not None else None
    b = solver._as_dev(drift) if drift is not None else None
    dev = solver.device
    v = t.empty((K, M), device=dev)
    dv = t.empty((K, M, n), device=dev) if want_dv else None
    c = t.empty((K, M), device=dev)
    iters = t.zeros(K, dtype=t.int32, device=dev)
    eps = t.empty((K, max_iter), dtype=t.float64, device=dev)
    dsup = t.empty((K, max_iter), dtype=t.float64, device=dev)
    tube = t.empty(M, device=dev)
    ptr = lambda a: C.c_void_p(a.data_ptr()) if a is not None else None
    solver._check(solver.L.hjmc_picard_solve(
        solver.h, ptr(x), ptr(q), qid_base, M, ptr(b), float(tol), int(max_iter), ptr(v), ptr(dv),
        ptr(c), ptr(iters), ptr(eps), ptr(dsup), ptr(tube), solver._stream()))
    eps_h = eps.cpu().numpy()
    it = iters.cpu().numpy().astype(np.int64)
    conv = np.array([it[j] > 0 and eps_h[j, it[j] - 1] < tol for j in range(K)])
    return {"v": v, "dv": dv, "c": c, "iters": it, "eps": eps_h, "d_sup": dsup.cpu().numpy(),
            "tube": tube, "converged": conv}


def solve_adaptive_resident(solver, x, tol: float, max_iter: int, qid_base: int = 0, qid=None,
                            drift=None, group=None, graph: bool = False, want_dv: bool = True):
    """Algorithm 1 with its stopping test for a sharded slice, device-resident: every iterate is
    {hjmc_picard_dev_pass → all-reduce of the [3][K] partials on the stream (NCCL through
    torch.distributed when `group` is given: rows 0–1 summed, row 2 maxed) →
    hjmc_picard_dev_decide}, enqueued max_iter times with no host round trip (retired horizons'
    passes exit at once); graph=True captures the whole loop, collectives included, into one
    CUDA graph and replays it. With one process it equals solve_adaptive_device bit for bit.
    Returns the dict of solve_adaptive_device (v, dv, c, iters, eps, d_sup, tube, converged)."""
    t = solver.torch
    cfg = solver.cfg
    x = solver._as_query(x)
    M, K, n = x.shape[0], cfg.K, cfg.n
    q = solver._as_dev(qid, t.int32) if qid is not None else None
    b = solver._as_dev(drift) if drift is not None else None
    dev = solver.device
    v = t.empty((K, M), device=dev)
    dv = t.empty((K, M, n), device=dev) if want_dv else None
    c = t.empty((K, M), device=dev)
    iters = t.zeros(K, dtype=t.int32, device=dev)
    eps = t.empty((K, max_iter), dtype=t.float64, device=dev)
    dsup = t.empty((K, max_iter), dtype=t.float64, device=dev)
    red = t.empty((3, K), dtype=t.float64, device=dev)
    tube = t.empty(M, device=dev)
    L = solver.L
    ptr = lambda a: C.c_void_p(a.data_ptr()) if a is not None else None
    solver._check(L.hjmc_picard_dev_begin(solver.h, ptr(x), ptr(q), qid_base, M, ptr(b),
                                          int(max_iter), ptr(iters), ptr(eps), ptr(dsup),
                                          solver._stream()))

    def body():
        import torch.distributed as dist

        stream = solver._stream()
        for _ in range(max_iter):
            solver._check(L.hjmc_picard_dev_pass(solver.h, ptr(v), ptr(dv), ptr(c), ptr(red),
                                                 stream))
            if group is not None:
                dist.all_reduce(red[:2], op=dist.ReduceOp.SUM, group=group)
                dist.all_reduce(red[2], op=dist.ReduceOp.MAX, group=group)
            solver._check(L.hjmc_picard_dev_decide(solver.h, ptr(red), float(tol), ptr(iters),
                                                   ptr(eps), ptr(dsup), stream))

    if graph:
        t.cuda.synchronize(dev)
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g):
            body()
        g.replay()
    else:
        body()
    solver._check(L.hjmc_tube(solver.h, ptr(x), M, ptr(v), ptr(tube), solver._stream()))
    eps_h = eps.cpu().numpy()
    it = iters.cpu().numpy().astype(np.int64)
    conv = np.array([it[j] > 0 and eps_h[j, it[j] - 1] < tol for j in range(K)])
    return {"v": v, "dv": dv, "c": c, "iters": it, "eps": eps_h, "d_sup": dsup.cpu().numpy(),
            "tube": tube, "converged": conv}

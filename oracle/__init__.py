"""TEST INFRASTRUCTURE ONLY — the CPU oracle (plain C, double precision) and its ctypes wrapper.

Who may import this: tests/, __graft_entry__.smoke(), and bench.py's cpu_baseline /
--impl reference legs. The product package (paper_2605_18566_b200) never imports it and
fails loudly when its own CUDA library is missing.

The oracle shares no code with the CUDA path; see hjmc_oracle.h for the pins of each function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "hjmc_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

SYSTEMS = {"quadratic": 0, "dubins_rel": 1, "rocket6": 2, "dubins_pairs": 3, "rocket3": 4,
           "double_integrator": 5, "multiagent": 6}
TARGETS = {"quad_bowl": 0, "disk": 1, "rel_disk6": 2, "pair_union": 3, "linear": 4, "const": 5,
           "pursuit_min": 6}
AVOIDS = {"none": 0, "disk": 1}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, OpenMP over independent queries)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", LIB, SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB


class _Problem(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("delta", C.c_double), ("T", C.c_double), ("K", C.c_int32),
        ("Kp", C.c_int32), ("N", C.c_uint32), ("seed", C.c_uint64),
        ("full_laplacian", C.c_int32), ("crn", C.c_int32), ("antithetic", C.c_int32),
        ("m0", C.c_double), ("c_min", C.c_double), ("c_max", C.c_double), ("tag", C.c_uint32),
        ("system", C.c_int32), ("n_sys_params", C.c_int32), ("sys_params", C.c_double * 8),
        ("target", C.c_int32), ("n_tgt_params", C.c_int32), ("tgt_params", C.c_double * 72),
        ("avoid", C.c_int32), ("avoid_params", C.c_double * 3), ("proposal", C.c_int32),
    ]


_lib = None


def build_sanitized(path: str = os.path.join(HERE, "liboracle_san.so")) -> str:
    """The same oracle compiled with -fsanitize=address,undefined (tools/sanitize_oracle.sh runs
    the CPU suite against it with HJMC_ORACLE_LIB=<path> and libasan preloaded)."""
    cmd = ["gcc", "-O1", "-g", "-std=c11", "-fopenmp", "-fPIC", "-shared",
           "-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
           "-fno-omit-frame-pointer", "-o", path, SRC, "-lm"]
    subprocess.run(cmd, check=True)
    return path


def lib():
    global _lib
    if _lib is None:
        path = os.environ.get("HJMC_ORACLE_LIB")
        if not path:
            build()
        L = C.CDLL(path or LIB)
        dp, fp, up = C.POINTER(C.c_double), C.POINTER(C.c_float), C.POINTER(C.c_uint32)
        pp = C.POINTER(_Problem)
        L.orc_philox4x32_10.argtypes = [up, up, up]
        L.orc_sample_normals.argtypes = [pp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, dp, up]
        L.orc_target_g.argtypes = [pp, dp]
        L.orc_target_g.restype = C.c_double
        L.orc_target_dg.argtypes = [pp, dp, dp]
        L.orc_avoid_l.argtypes = [pp, dp]
        L.orc_avoid_l.restype = C.c_double
        L.orc_hamiltonian.argtypes = [pp, dp, dp]
        L.orc_hamiltonian.restype = C.c_double
        L.orc_gamma.argtypes = [pp, dp, dp]
        L.orc_gamma.restype = C.c_double
        L.orc_phi.argtypes = [pp, dp, dp, C.c_uint32, C.c_double, C.c_double, C.c_uint32,
                              C.c_uint32, dp, dp, dp, dp]
        L.orc_phi.restype = C.c_int
        L.orc_solve_slice.argtypes = [pp, fp, fp, up, C.c_uint32, C.c_int64, dp, dp, dp, dp, dp,
                                      dp, dp, dp, C.c_int32]
        L.orc_solve_slice.restype = C.c_int
        L.orc_residual_partials.argtypes = [dp, dp, C.c_int32, C.c_int32, C.c_int64, dp]
        L.orc_picard_adaptive.argtypes = [pp, fp, up, C.c_uint32, C.c_int64, C.c_double, C.c_int32,
                                          dp, dp, dp, dp, C.c_int32]
        L.orc_picard_adaptive.restype = C.c_int
        L.orc_phi_batch.argtypes = [pp, fp, C.POINTER(C.c_int64), up, dp, dp, up, up, C.c_int64,
                                    dp, dp, C.c_int32]
        L.orc_phi_batch.restype = C.c_int
        L.orc_tube.argtypes = [pp, fp, C.c_int64, dp, dp]
        L.orc_tube.restype = None
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


@dataclass
class Problem:
    n: int
    delta: float = 0.05
    T: float = 0.5
    K: int = 1
    Kp: int = 1
    N: int = 4096
    seed: int = 0x5EED000000000001
    visc: str = "paper"
    crn: bool = True
    antithetic: bool = False
    m0: float = 1e-3
    c_min: float = 0.05
    c_max: float = 20.0
    tag: int = 0
    system: str = "quadratic"
    sys_params: tuple = ()
    target: str = "quad_bowl"
    tgt_params: tuple = ()
    avoid: str = "none"
    avoid_params: tuple = ()
    proposal: str = "plain"            # "plain" | "laplace" (R28)

    @classmethod
    def from_preset(cls, p, **kw):
        d = dict(n=p.n, delta=p.delta, T=p.T, K=p.K, Kp=p.Kp, N=p.N, seed=p.seed, visc=p.visc,
                 crn=p.crn, antithetic=p.antithetic, m0=p.m0, c_min=p.c_min, c_max=p.c_max,
                 tag=p.tag, system=p.system, sys_params=tuple(p.sys_params), target=p.target,
                 tgt_params=tuple(p.tgt_params), avoid=getattr(p, "avoid", "none"),
                 avoid_params=tuple(getattr(p, "avoid_params", ())),
                 proposal=getattr(p, "proposal", "plain"))
        d.update(kw)
        return cls(**d)

    def struct(self) -> _Problem:
        s = _Problem()
        s.n, s.delta, s.T, s.K, s.Kp, s.N = self.n, self.delta, self.T, self.K, self.Kp, self.N
        s.seed = self.seed
        s.full_laplacian = 1 if self.visc == "full" else 0
        s.crn, s.antithetic = int(self.crn), int(self.antithetic)
        s.m0, s.c_min, s.c_max, s.tag = self.m0, self.c_min, self.c_max, self.tag
        s.system = SYSTEMS[self.system]
        s.n_sys_params = len(self.sys_params)
        for i, v in enumerate(self.sys_params):
            s.sys_params[i] = v
        s.target = TARGETS[self.target]
        s.n_tgt_params = len(self.tgt_params)
        for i, v in enumerate(self.tgt_params):
            s.tgt_params[i] = v
        s.avoid = AVOIDS[self.avoid]
        s.proposal = {"plain": 0, "laplace": 1}[self.proposal]
        for i, v in enumerate(self.avoid_params):
            s.avoid_params[i] = v
        return s

    @property
    def delta_eff(self) -> float:
        return 2.0 * self.delta if self.visc == "full" else self.delta


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (C.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return [int(v) for v in o]


def normals(P: Problem, qid: int, jw: int, kw: int, i0: int, count: int, raw: bool = False):
    s = P.struct()
    nq = (P.n + 3) // 4 + 1                      # blocks a sample can touch (R19 grouping)
    z = np.zeros((count, P.n))
    r = np.zeros((count, 4 * nq), dtype=np.uint32)
    for t in range(count):
        zt = np.zeros(P.n)
        rt = np.zeros(4 * nq, dtype=np.uint32)
        lib().orc_sample_normals(C.byref(s), qid, jw, kw, i0 + t, _dp(zt),
                                 rt.ctypes.data_as(C.POINTER(C.c_uint32)))
        z[t], r[t] = zt, rt
    return (z, r) if raw else z


def g(P: Problem, y) -> float:
    y = np.ascontiguousarray(y, dtype=np.float64)
    return lib().orc_target_g(C.byref(P.struct()), _dp(y))


def dg(P: Problem, x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    o = np.zeros(P.n)
    lib().orc_target_dg(C.byref(P.struct()), _dp(x), _dp(o))
    return o


def avoid_l(P: Problem, x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().orc_avoid_l(C.byref(P.struct()), _dp(x))


def hamiltonian(P: Problem, x, p) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    return lib().orc_hamiltonian(C.byref(P.struct()), _dp(x), _dp(p))


def gamma(P: Problem, x, p) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    return lib().orc_gamma(C.byref(P.struct()), _dp(x), _dp(p))


def phi(P: Problem, x, c: float, tau: float, qid: int = 0, jw: int = 1, kw: int = 0, drift=None):
    """One Φ pass for one query. Returns (v, dv[n], diag[6], se_dv[n])."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    b = None if drift is None else np.ascontiguousarray(drift, dtype=np.float64)
    v = np.zeros(1)
    dv = np.zeros(P.n)
    diag = np.zeros(6)
    se = np.zeros(P.n)
    st = lib().orc_phi(C.byref(P.struct()), _dp(x), _dp(b), qid, c, tau, jw, kw, _dp(v), _dp(dv),
                       _dp(diag), _dp(se))
    if st == 1:
        raise MemoryError("oracle phi: allocation failed")
    return float(v[0]), dv, diag, se


def phi_batch(P: Problem, x, c, tau: float, qid_base: int = 0, jw: int = 1, kw: int = 0,
              drift=None, qids=None):
    """Φ over M queries (sequential loop of orc_phi). Returns (v[M], dv[M][n])."""
    x = np.asarray(x, dtype=np.float64)
    M = x.shape[0]
    c = np.broadcast_to(np.asarray(c, dtype=np.float64), (M,))
    v = np.zeros(M)
    dv = np.zeros((M, P.n))
    for m in range(M):
        q = int(qids[m]) if qids is not None else qid_base + m
        b = None if drift is None else drift[m]
        v[m], dv[m], _, _ = phi(P, x[m], float(c[m]), tau, q, jw, kw, b)
    return v, dv


def phi_items(P: Problem, x, xi, qid, c, tau, jw, kw, nthreads: int = 0, want_dv: bool = True):
    """Φ at independent items i: query x[xi[i]] (the fp32 array, converted to double), global
    id qid[i], frozen coefficient c[i], time-to-go tau[i], counter tags jw[i], kw[i] — a plain
    OpenMP loop of orc_phi (orc_phi_batch). Returns (v[count], dv[count][n] or None)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    cnt = len(xi)
    arr = lambda a, dt: np.ascontiguousarray(np.broadcast_to(np.asarray(a), (cnt,)), dtype=dt)
    xi_, q_ = arr(xi, np.int64), arr(qid, np.uint32)
    c_, t_ = arr(c, np.float64), arr(tau, np.float64)
    j_, k_ = arr(jw, np.uint32), arr(kw, np.uint32)
    v = np.zeros(cnt)
    dv = np.zeros((cnt, P.n)) if want_dv else None
    up = C.POINTER(C.c_uint32)
    st = lib().orc_phi_batch(C.byref(P.struct()), x.ctypes.data_as(C.POINTER(C.c_float)),
                             xi_.ctypes.data_as(C.POINTER(C.c_int64)), q_.ctypes.data_as(up),
                             _dp(c_), _dp(t_), j_.ctypes.data_as(up), k_.ctypes.data_as(up), cnt,
                             _dp(v), _dp(dv), nthreads)
    if st == 1:
        raise MemoryError("oracle phi: allocation failed")
    return v, dv


def solve_slice(P: Problem, x, drift=None, qid_base: int = 0, qids=None, nthreads: int = 0):
    """Algorithm 1 over all horizons for the fp32 queries x[M][n]; returns a dict of float64."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    M = x.shape[0]
    n, K, Kp = P.n, P.K, P.Kp
    out = {
        "v": np.zeros(M), "dv": np.zeros((M, n)), "c": np.zeros(M), "tube": np.zeros(M),
        "vhist": np.zeros((K, Kp, M)), "chist": np.zeros((K, Kp, M)), "g0": np.zeros(M),
        "dvhist": np.zeros((K, Kp, M, n)),
    }
    b = None if drift is None else np.ascontiguousarray(drift, dtype=np.float32)
    q = None if qids is None else np.ascontiguousarray(qids, dtype=np.uint32)
    st = lib().orc_solve_slice(
        C.byref(P.struct()), x.ctypes.data_as(C.POINTER(C.c_float)),
        b.ctypes.data_as(C.POINTER(C.c_float)) if b is not None else None,
        q.ctypes.data_as(C.POINTER(C.c_uint32)) if q is not None else None,
        qid_base, M, _dp(out["v"]), _dp(out["dv"]), _dp(out["c"]), _dp(out["tube"]),
        _dp(out["vhist"]), _dp(out["chist"]), _dp(out["g0"]), _dp(out["dvhist"]), nthreads)
    out["status"] = st
    return out


def picard_adaptive(P: Problem, x, tol: float, max_iter: int, qid_base: int = 0, qids=None,
                    nthreads: int = 0):
    """Algorithm 1 with the convergence test, per horizon. Returns v [K][M], iters [K],
    eps [K][max_iter], d_sup [K][max_iter], tube [M] (orc_tube: running min with the BRAT
    clamp)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    M, K = x.shape[0], P.K
    v = np.zeros((K, M))
    iters = np.zeros(K)
    eps = np.zeros((K, max_iter))
    dsup = np.zeros((K, max_iter))
    q = None if qids is None else np.ascontiguousarray(qids, dtype=np.uint32)
    st = lib().orc_picard_adaptive(C.byref(P.struct()), x.ctypes.data_as(C.POINTER(C.c_float)),
                                   q.ctypes.data_as(C.POINTER(C.c_uint32)) if q is not None else None,
                                   qid_base, M, tol, max_iter, _dp(v), _dp(iters), _dp(eps),
                                   _dp(dsup), nthreads)
    tube = np.zeros(M)
    lib().orc_tube(C.byref(P.struct()), x.ctypes.data_as(C.POINTER(C.c_float)), M, _dp(v), _dp(tube))
    return {"v": v, "iters": iters.astype(int), "eps": eps, "d_sup": dsup, "tube": tube,
            "status": st}


def gamma_sensitivity(P: Problem, x, p, rel: float = 1e-6) -> float:
    """‖∇_p Γ(x, p)‖₂ by central differences (steps rel·max(|p|, m0)); used by the parity tests
    to bound how far c = Γ(x, Dv) may move when Dv carries a small relative error."""
    x = np.asarray(x, dtype=np.float64)
    p = np.asarray(p, dtype=np.float64)
    h = rel * max(np.linalg.norm(p), P.m0)
    g = np.zeros(P.n)
    for d in range(P.n):
        e = np.zeros(P.n)
        e[d] = h
        g[d] = (gamma(P, x, p + e) - gamma(P, x, p - e)) / (2 * h)
    return float(np.linalg.norm(g))


def residual_partials(vhist, g0):
    vhist = np.ascontiguousarray(vhist, dtype=np.float64)
    g0 = np.ascontiguousarray(g0, dtype=np.float64)
    K, Kp, M = vhist.shape
    out = np.zeros((K, Kp, 2))
    lib().orc_residual_partials(_dp(vhist), _dp(g0), K, Kp, M, _dp(out))
    return out


def max_threads() -> int:
    return lib().orc_max_threads()

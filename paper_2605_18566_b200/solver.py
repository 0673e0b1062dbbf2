"""Python binding of libhjmc (argument marshalling only; every step runs in the CUDA kernels).

PyTorch supplies device memory and the current CUDA stream; the library computes.
Names follow include/hjmc.h, which cites the paper passage behind each entry point.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .inputs import Preset


@dataclass
class SolverConfig:
    n: int
    delta: float
    T: float = 1.0
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
    device: int = 0
    sync_check: bool = False
    skip_stationary: bool = False
    reuse_passes: bool = False   # HJMC_FLAG_REUSE_PASSES (exact pass memo under CRN)
    speculate: bool = False      # HJMC_FLAG_SPECULATE_CLAMPS (memoize the opposite clamp too)
    system: str = "quadratic"
    sys_params: tuple = ()
    target: str = "quad_bowl"
    tgt_params: tuple = ()
    avoid: str = "none"
    avoid_params: tuple = ()
    proposal: str = "plain"      # "plain" | "laplace" (R28)

    @classmethod
    def from_preset(cls, p: Preset, **kw) -> "SolverConfig":
        d = dict(n=p.n, delta=p.delta, T=p.T, K=p.K, Kp=p.Kp, N=p.N, seed=p.seed, visc=p.visc,
                 crn=p.crn, antithetic=p.antithetic, m0=p.m0, c_min=p.c_min, c_max=p.c_max,
                 tag=p.tag, system=p.system, sys_params=tuple(p.sys_params), target=p.target,
                 tgt_params=tuple(p.tgt_params), avoid=p.avoid, avoid_params=tuple(p.avoid_params),
                 proposal=p.proposal)
        d.update(kw)
        return cls(**d)

    def struct(self) -> _lib.Config:
        c = _lib.Config()
        c.n, c.delta, c.T, c.K, c.Kp, c.N = self.n, self.delta, self.T, self.K, self.Kp, self.N
        c.seed = self.seed
        c.visc = _lib.VISC[self.visc]
        c.crn, c.antithetic = int(self.crn), int(self.antithetic)
        c.m0, c.c_min, c.c_max, c.tag, c.device = self.m0, self.c_min, self.c_max, self.tag, self.device
        c.proposal = _lib.PROPOSALS[self.proposal]
        c.flags = (_lib.FLAG_SYNC_CHECK if self.sync_check else 0) | (
            _lib.FLAG_SKIP_STATIONARY if self.skip_stationary else 0) | (
            _lib.FLAG_REUSE_PASSES if self.reuse_passes else 0) | (
            _lib.FLAG_SPECULATE_CLAMPS if self.speculate else 0)
        return c


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _floats(vals):
    arr = (C.c_float * max(1, len(vals)))(*[float(v) for v in vals])
    return arr, len(vals)


class Solver:
    """One libhjmc handle: a configured system + target on one CUDA device."""

    def __init__(self, cfg: SolverConfig):
        import torch

        self.torch = torch
        self.cfg = cfg
        self.L = _lib.load()
        self.device = torch.device("cuda", cfg.device)
        h = C.c_void_p()
        s = cfg.struct()
        self._check(self.L.hjmc_create(C.byref(s), C.byref(h)), None)
        self.h = h
        arr, np_ = _floats(cfg.sys_params)
        self._check(self.L.hjmc_set_dynamics(self.h, _lib.SYSTEMS[cfg.system], arr, np_))
        arr, np_ = _floats(cfg.tgt_params)
        self._check(self.L.hjmc_set_target(self.h, _lib.TARGETS[cfg.target], arr, np_))
        if cfg.avoid != "none":
            arr, np_ = _floats(cfg.avoid_params)
            self._check(self.L.hjmc_set_avoid(self.h, _lib.AVOIDS[cfg.avoid], arr, np_))

    # -- plumbing --------------------------------------------------------------------------
    def _check(self, rc, h="self"):
        if rc != 0:
            hh = self.h if h == "self" else h
            msg = self.L.hjmc_last_error(hh)
            raise _lib.HjmcError(rc, msg.decode() if msg else "")

    def close(self):
        if getattr(self, "h", None):
            self.L.hjmc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def _as_dev(self, a, dtype=None):
        t = self.torch
        dtype = dtype or t.float32
        if isinstance(a, t.Tensor):
            a = a.to(device=self.device, dtype=dtype)
        else:
            a = t.as_tensor(np.asarray(a), dtype=dtype, device=self.device)
        return a.contiguous()

    def _as_query(self, x):
        x = self._as_dev(x)
        if x.dim() != 2 or x.shape[1] != self.cfg.n:
            raise ValueError(f"queries must have shape (M, {self.cfg.n}), got {tuple(x.shape)}")
        return x

    # -- entry points ------------------------------------------------------------------------
    def value_grad(self, x, c, tau: float, j_tag: int = 1, k_tag: int = 0, qid_base: int = 0,
                   qid=None, drift=None, want_dv: bool = True):
        """One Φ pass at frozen per-query c (hjmc_value_grad). Returns (v[M], dv[M][n])."""
        t = self.torch
        x = self._as_query(x)
        M = x.shape[0]
        c = self._as_dev(c) if c is not None else None
        if c is not None and tuple(c.shape) != (M,):
            raise ValueError(f"c must have shape ({M},), got {tuple(c.shape)}")
        drift = self._as_dev(drift) if drift is not None else None
        if drift is not None and tuple(drift.shape) != tuple(x.shape):
            raise ValueError(f"drift must have the queries' shape {tuple(x.shape)}")
        q = self._as_dev(qid, t.int32) if qid is not None else None
        if q is not None and tuple(q.shape) != (M,):
            raise ValueError(f"qid must have shape ({M},), got {tuple(q.shape)}")
        v = t.empty(M, device=self.device)
        dv = t.empty((M, self.cfg.n), device=self.device) if want_dv else None
        self._check(self.L.hjmc_value_grad(self.h, _ptr(x), _ptr(c), _ptr(q), qid_base, M,
                                           float(tau), j_tag, k_tag, _ptr(drift), _ptr(v),
                                           _ptr(dv), self._stream()))
        return v, dv

    def alloc_result(self, M: int, hist: bool = True):
        t, n, K, Kp = self.torch, self.cfg.n, self.cfg.K, self.cfg.Kp
        e = lambda *s: t.empty(s, device=self.device)
        r = {"v": e(M), "dv": e(M, n), "c": e(M), "tube": e(M), "g0": e(M)}
        if hist:
            r["vhist"] = e(K, Kp, M)
            r["chist"] = e(K, Kp, M)
        return r

    def _shapes(self, M: int) -> dict:
        n, K, Kp = self.cfg.n, self.cfg.K, self.cfg.Kp
        return {"v": (M,), "dv": (M, n), "c": (M,), "tube": (M,), "g0": (M,),
                "vhist": (K, Kp, M), "chist": (K, Kp, M)}

    def _check_out(self, out: dict, M: int):
        """Caller-provided output buffers: the C-ABI writes through raw pointers, so shape,
        dtype, device and contiguity are checked here rather than trusted."""
        t = self.torch
        for k, shape in self._shapes(M).items():
            a = out.get(k)
            if a is None:
                continue
            if (tuple(a.shape) != shape or a.dtype != t.float32 or a.device != self.device
                    or not a.is_contiguous()):
                raise ValueError(f"out[{k!r}] must be a contiguous float32 tensor of shape "
                                 f"{shape} on {self.device}, got {tuple(a.shape)} {a.dtype} "
                                 f"{a.device}")

    def solve_slice(self, x, qid_base: int = 0, qid=None, drift=None, out=None, hist: bool = True):
        """Algorithm 1 over all horizons + tube (hjmc_solve_slice). Returns a dict of tensors."""
        t = self.torch
        x = self._as_query(x)
        M = x.shape[0]
        drift = self._as_dev(drift) if drift is not None else None
        if drift is not None and tuple(drift.shape) != tuple(x.shape):
            raise ValueError(f"drift must have the queries' shape {tuple(x.shape)}")
        q = self._as_dev(qid, t.int32) if qid is not None else None
        if q is not None and tuple(q.shape) != (M,):
            raise ValueError(f"qid must have shape ({M},), got {tuple(q.shape)}")
        if out is None:
            out = self.alloc_result(M, hist)
        else:
            self._check_out(out, M)
        res = _lib.Result(*[C.c_void_p(out[k].data_ptr()) if out.get(k) is not None else None
                            for k in ("v", "dv", "c", "tube", "vhist", "chist", "g0")])
        self._check(self.L.hjmc_solve_slice(self.h, _ptr(x), _ptr(q), qid_base, M, _ptr(drift),
                                            C.byref(res), self._stream()))
        return out

    def solve_slice_host(self, x: np.ndarray, qid_base: int = 0, drift=None, out=None,
                         hist: bool = True, qid=None):
        """End-to-end call with HOST arrays (hjmc_solve_slice_host); synchronous. qid: optional
        host array of explicit global query ids (uint32/int32, shape (M,))."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        if x.ndim != 2 or x.shape[1] != self.cfg.n:
            raise ValueError(f"queries must have shape (M, {self.cfg.n}), got {x.shape}")
        M, n, K, Kp = x.shape[0], self.cfg.n, self.cfg.K, self.cfg.Kp
        if out is None:
            out = {"v": np.empty(M, np.float32), "dv": np.empty((M, n), np.float32),
                   "c": np.empty(M, np.float32), "tube": np.empty(M, np.float32),
                   "g0": np.empty(M, np.float32)}
            if hist:
                out["vhist"] = np.empty((K, Kp, M), np.float32)
                out["chist"] = np.empty((K, Kp, M), np.float32)
        keys = ("v", "dv", "c", "tube", "vhist", "chist", "g0")
        # the C-ABI copies through raw host pointers: check every buffer's shape and layout
        for k, shape in self._shapes(M).items():
            a = out.get(k)
            if a is None:
                continue
            is_t = hasattr(a, "data_ptr")
            dt_ok = (a.dtype == self.torch.float32) if is_t else (a.dtype == np.float32)
            contig = a.is_contiguous() if is_t else a.flags["C_CONTIGUOUS"]
            on_host = (a.device.type == "cpu") if is_t else True
            if tuple(a.shape) != shape or not dt_ok or not contig or not on_host:
                raise ValueError(f"out[{k!r}] must be a contiguous host float32 array of shape "
                                 f"{shape}, got {tuple(a.shape)} {a.dtype}")
        res = _lib.Result(*[C.c_void_p(_host_ptr(out[k])) if out.get(k) is not None else None
                            for k in keys])
        b = None if drift is None else np.ascontiguousarray(drift, dtype=np.float32)
        if b is not None and b.shape != x.shape:
            raise ValueError(f"drift must have the queries' shape {x.shape}")
        q = None
        if qid is not None:
            q = qid if hasattr(qid, "data_ptr") else np.ascontiguousarray(qid).astype(np.uint32)
            if tuple(q.shape) != (M,) or (hasattr(q, "is_contiguous") and not q.is_contiguous()):
                raise ValueError(f"qid must be a contiguous host array of shape ({M},)")
        self._check(self.L.hjmc_solve_slice_host(
            self.h, C.c_void_p(_host_ptr(x)), C.c_void_p(_host_ptr(q)) if q is not None else None,
            qid_base, M, C.c_void_p(_host_ptr(b)) if b is not None else None, C.byref(res)))
        return out

    def eval_target(self, x):
        x = self._as_dev(x)
        M = x.shape[0]
        g = self.torch.empty(M, device=self.device)
        dg = self.torch.empty((M, self.cfg.n), device=self.device)
        self._check(self.L.hjmc_eval_target(self.h, _ptr(x), M, _ptr(g), _ptr(dg), self._stream()))
        return g, dg

    def eval_hamiltonian(self, x, p):
        x, p = self._as_dev(x), self._as_dev(p)
        M = x.shape[0]
        H = self.torch.empty(M, device=self.device)
        c = self.torch.empty(M, device=self.device)
        self._check(self.L.hjmc_eval_hamiltonian(self.h, _ptr(x), _ptr(p), M, _ptr(H), _ptr(c),
                                                 self._stream()))
        return H, c

    def debug_normals(self, qid: int, jw: int, kw: int, i0: int, count: int, raw: bool = False):
        t = self.torch
        n = self.cfg.n
        z = t.empty((count, n), device=self.device)
        r = t.zeros((count, 4 * ((n + 3) // 4 + 1)), dtype=t.int32, device=self.device) if raw else None
        self._check(self.L.hjmc_debug_normals(self.h, qid, jw, kw, i0, count, _ptr(z), _ptr(r),
                                              self._stream()))
        return (z, r) if raw else z

    def check(self):
        """Synchronise and raise HjmcError(ENUMERIC) on a recorded numerical failure."""
        self._check(self.L.hjmc_check(self.h, self._stream()))

    def pass_count(self) -> int:
        """Φ passes executed since the previous call (synchronises)."""
        v = C.c_uint64()
        self._check(self.L.hjmc_pass_count(self.h, self._stream(), C.byref(v)))
        return int(v.value)

    def last_bad_query(self) -> int:
        return int(self.L.hjmc_last_bad_query(self.h))


def _host_ptr(a) -> int:
    if a is None:
        return 0
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def residual_partials(vhist: np.ndarray, g0: np.ndarray) -> np.ndarray:
    """(num, den) per (j, k) for ε_j(k) = sqrt(num/den) (hjmc_residual_partials)."""
    L = _lib.load()
    vhist = np.ascontiguousarray(vhist, dtype=np.float32)
    g0 = np.ascontiguousarray(g0, dtype=np.float32)
    K, Kp, M = vhist.shape
    out = np.zeros((K, Kp, 2), dtype=np.float64)
    rc = L.hjmc_residual_partials(C.c_void_p(vhist.ctypes.data), C.c_void_p(g0.ctypes.data), K,
                                  Kp, M, C.c_void_p(out.ctypes.data))
    if rc != 0:
        raise _lib.HjmcError(rc, "residual_partials")
    return out


def residual_eps(partials: np.ndarray) -> np.ndarray:
    """ε = sqrt(num / max(den, 1e-300)) per (num, den) pair (hjmc_residual_eps, R11)."""
    L = _lib.load()
    part = np.ascontiguousarray(partials, dtype=np.float64)
    if part.shape[-1] != 2:
        raise ValueError("partials must end in a (num, den) axis")
    out = np.empty(part.shape[:-1], dtype=np.float64)
    rc = L.hjmc_residual_eps(C.c_void_p(part.ctypes.data), out.size, C.c_void_p(out.ctypes.data))
    if rc != 0:
        raise _lib.HjmcError(rc, "residual_eps")
    return out


def supported(target: str, n: int) -> bool:
    return bool(_lib.load().hjmc_supported(_lib.TARGETS[target], n))

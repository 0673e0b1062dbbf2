"""ctypes declarations of libhjmc's C-ABI (include/hjmc.h). Marshalling only: no arithmetic.

The library is loaded from this package directory. If it is missing the import of the
binding raises — there is no CPU or pure-Python fallback for any step of the path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhjmc.so")

HJMC_OK, HJMC_EINVAL, HJMC_ENUMERIC, HJMC_ECUDA, HJMC_EUNSUPPORTED, HJMC_ENOMEM = range(6)
ERROR_NAMES = {0: "OK", 1: "EINVAL", 2: "ENUMERIC", 3: "ECUDA", 4: "EUNSUPPORTED", 5: "ENOMEM"}
SYSTEMS = {"quadratic": 0, "dubins_rel": 1, "rocket6": 2, "dubins_pairs": 3, "rocket3": 4,
           "double_integrator": 5, "multiagent": 6}
TARGETS = {"quad_bowl": 0, "disk": 1, "rel_disk6": 2, "pair_union": 3, "linear": 4, "const": 5,
           "pursuit_min": 6}
AVOIDS = {"none": 0, "disk": 1}
VISC = {"paper": 0, "full": 1}
FLAG_SYNC_CHECK = 1
FLAG_SKIP_STATIONARY = 2
FLAG_REUSE_PASSES = 4
FLAG_SPECULATE_CLAMPS = 8
PROPOSALS = {"plain": 0, "laplace": 1}

EXPORTS = [
    "hjmc_config_defaults", "hjmc_create", "hjmc_destroy", "hjmc_set_dynamics", "hjmc_set_target",
    "hjmc_supported", "hjmc_value_grad", "hjmc_solve_slice", "hjmc_solve_slice_host",
    "hjmc_eval_target", "hjmc_eval_hamiltonian", "hjmc_debug_normals", "hjmc_check",
    "hjmc_last_bad_query", "hjmc_last_error", "hjmc_residual_partials", "hjmc_version",
    "hjmc_pass_count", "hjmc_picard_begin", "hjmc_picard_pass", "hjmc_picard_solve",
    "hjmc_set_avoid", "hjmc_picard_decide", "hjmc_residual_eps", "hjmc_tube",
    "hjmc_contraction_constant", "hjmc_contraction_report", "hjmc_picard_dev_begin",
    "hjmc_picard_dev_pass", "hjmc_picard_dev_decide",
]


class Config(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("delta", C.c_float), ("T", C.c_float), ("K", C.c_int32),
        ("Kp", C.c_int32), ("N", C.c_uint32), ("seed", C.c_uint64), ("visc", C.c_int32),
        ("crn", C.c_int32), ("antithetic", C.c_int32), ("m0", C.c_float), ("c_min", C.c_float),
        ("c_max", C.c_float), ("tag", C.c_uint32), ("device", C.c_int32), ("flags", C.c_uint32),
        ("proposal", C.c_int32),
    ]


class Result(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("v", "dv", "c", "tube", "vhist", "chist", "g0")]


class HjmcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"hjmc error {ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def load(path: str = LIB_PATH):
    """Load libhjmc.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2605_18566_b200.build` "
            "(the hot path has no CPU fallback)")
    L = C.CDLL(path)
    vp, i64, u32, fp = C.c_void_p, C.c_int64, C.c_uint32, C.c_float
    L.hjmc_config_defaults.argtypes = [C.POINTER(Config)]
    L.hjmc_config_defaults.restype = None
    L.hjmc_create.argtypes = [C.POINTER(Config), C.POINTER(vp)]
    L.hjmc_destroy.argtypes = [vp]
    L.hjmc_destroy.restype = None
    L.hjmc_set_dynamics.argtypes = [vp, C.c_int32, C.POINTER(C.c_float), C.c_int32]
    L.hjmc_set_target.argtypes = [vp, C.c_int32, C.POINTER(C.c_float), C.c_int32]
    L.hjmc_supported.argtypes = [C.c_int32, C.c_int32]
    L.hjmc_value_grad.argtypes = [vp, vp, vp, vp, u32, i64, fp, u32, u32, vp, vp, vp, vp]
    L.hjmc_solve_slice.argtypes = [vp, vp, vp, u32, i64, vp, C.POINTER(Result), vp]
    L.hjmc_solve_slice_host.argtypes = [vp, vp, vp, u32, i64, vp, C.POINTER(Result)]
    L.hjmc_eval_target.argtypes = [vp, vp, i64, vp, vp, vp]
    L.hjmc_eval_hamiltonian.argtypes = [vp, vp, vp, i64, vp, vp, vp]
    L.hjmc_debug_normals.argtypes = [vp, u32, u32, u32, u32, u32, vp, vp, vp]
    L.hjmc_check.argtypes = [vp, vp]
    L.hjmc_last_bad_query.argtypes = [vp]
    L.hjmc_last_bad_query.restype = i64
    L.hjmc_last_error.argtypes = [vp]
    L.hjmc_last_error.restype = C.c_char_p
    L.hjmc_residual_partials.argtypes = [vp, vp, C.c_int32, C.c_int32, i64, vp]
    L.hjmc_version.argtypes = []
    L.hjmc_pass_count.argtypes = [vp, vp, C.POINTER(C.c_uint64)]
    L.hjmc_set_avoid.argtypes = [vp, C.c_int32, C.POINTER(C.c_float), C.c_int32]
    L.hjmc_picard_begin.argtypes = [vp, vp, vp, u32, i64, vp, vp]
    L.hjmc_picard_pass.argtypes = [vp, C.c_int32, vp, vp, vp, vp, vp, vp]
    L.hjmc_picard_solve.argtypes = [vp, vp, vp, u32, i64, vp, C.c_double, C.c_int32, vp, vp, vp,
                                    vp, vp, vp, vp, vp]
    L.hjmc_picard_decide.argtypes = [vp, C.c_int32, C.c_double, vp, vp, vp, vp]
    L.hjmc_residual_eps.argtypes = [vp, i64, vp]
    L.hjmc_tube.argtypes = [vp, vp, i64, vp, vp, vp]
    dd = C.c_double
    L.hjmc_contraction_constant.argtypes = [dd] * 8
    L.hjmc_contraction_constant.restype = dd
    L.hjmc_contraction_report.argtypes = [vp, i64, dd, vp, vp]
    L.hjmc_picard_dev_begin.argtypes = [vp, vp, vp, u32, i64, vp, C.c_int32, vp, vp, vp, vp]
    L.hjmc_picard_dev_pass.argtypes = [vp, vp, vp, vp, vp, vp]
    L.hjmc_picard_dev_decide.argtypes = [vp, vp, dd, vp, vp, vp, vp]
    for name in EXPORTS:
        if not hasattr(L, name):
            raise RuntimeError(f"libhjmc.so lacks {name}")
    _lib = L
    return L

"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol that
include/hjmc.h declares, and its host-only entry points behave (no compute calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_18566_b200 import build, _lib

    build.build()
    return _lib.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hjmc.h")).read()
    return sorted(set(re.findall(r"HJMC_API\s+[\w\s\*]+?\b(hjmc_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared_symbols()
    assert len(names) >= 17
    for n in names:
        assert hasattr(lib, n), n
    from paper_2605_18566_b200 import _lib

    assert sorted(_lib.EXPORTS) == names


def test_only_api_symbols_exported():
    import subprocess

    from paper_2605_18566_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    text_syms = [l.split()[-1] for l in out.splitlines() if " T " in l]
    assert sorted(text_syms) == declared_symbols()


def test_config_defaults_and_version(lib):
    from paper_2605_18566_b200 import _lib

    c = _lib.Config()
    lib.hjmc_config_defaults(C.byref(c))
    assert (c.n, c.K, c.Kp, c.N, c.crn, c.antithetic) == (2, 1, 1, 4096, 1, 0)
    assert abs(c.m0 - 1e-3) < 1e-9 and c.c_min == pytest.approx(0.05) and c.c_max == 20.0
    assert c.seed == 0x5EED000000000001
    assert lib.hjmc_version() == 2


def test_supported_table(lib):
    T = {"quad_bowl": 0, "disk": 1, "rel_disk6": 2, "pair_union": 3}
    assert lib.hjmc_supported(T["disk"], 3) == 1
    assert lib.hjmc_supported(T["rel_disk6"], 6) == 1
    assert lib.hjmc_supported(T["pair_union"], 45) == 1
    assert lib.hjmc_supported(T["quad_bowl"], 2) == 1
    assert lib.hjmc_supported(T["rel_disk6"], 5) == 0
    assert lib.hjmc_supported(T["pair_union"], 7) == 0


def test_create_validation_without_gpu(lib):
    from paper_2605_18566_b200 import _lib

    c = _lib.Config()
    lib.hjmc_config_defaults(C.byref(c))
    h = C.c_void_p()
    for field, bad in (("delta", 0.0), ("T", -1.0), ("K", 0), ("Kp", 0), ("N", 0), ("n", 65),
                       ("c_min", 0.0), ("visc", 3)):
        cc = _lib.Config.from_buffer_copy(c)
        setattr(cc, field, bad)
        assert lib.hjmc_create(C.byref(cc), C.byref(h)) == _lib.HJMC_EINVAL, field
        assert not h.value
        assert lib.hjmc_last_error(None)
    cc = _lib.Config.from_buffer_copy(c)
    cc.c_min, cc.c_max = 5.0, 1.0
    assert lib.hjmc_create(C.byref(cc), C.byref(h)) == _lib.HJMC_EINVAL
    cc = _lib.Config.from_buffer_copy(c)
    cc.flags = 16                                  # no such flag bit
    assert lib.hjmc_create(C.byref(cc), C.byref(h)) == _lib.HJMC_EINVAL
    # every declared flag passes validation (then needs a device)
    cc.flags = (_lib.FLAG_SYNC_CHECK | _lib.FLAG_SKIP_STATIONARY | _lib.FLAG_REUSE_PASSES |
                _lib.FLAG_SPECULATE_CLAMPS)
    rcf = lib.hjmc_create(C.byref(cc), C.byref(h))
    assert rcf != _lib.HJMC_EINVAL
    if h.value:
        lib.hjmc_destroy(h)
        h = C.c_void_p()
    rc = lib.hjmc_create(C.byref(c), C.byref(h))
    import torch

    if not torch.cuda.is_available():
        assert rc == _lib.HJMC_ECUDA and not h.value
    else:
        assert rc == 0
        lib.hjmc_destroy(h)


def test_residual_partials_host_matches_oracle(lib, oracle_mod):
    from paper_2605_18566_b200.solver import residual_partials

    rng = np.random.default_rng(3)
    vhist = rng.normal(size=(3, 4, 50)).astype(np.float32)
    g0 = rng.normal(size=50).astype(np.float32)
    a = residual_partials(vhist, g0)
    b = oracle_mod.residual_partials(vhist.astype(np.float64), g0.astype(np.float64))
    np.testing.assert_allclose(a, b, rtol=1e-12)


def test_binding_fails_loudly_without_library(tmp_path):
    """No fallback: loading a missing library raises instead of degrading to CPU code."""
    from paper_2605_18566_b200 import _lib

    saved = _lib._lib
    try:
        _lib._lib = None
        with pytest.raises(RuntimeError, match="missing"):
            _lib.load(str(tmp_path / "missing.so"))
    finally:
        _lib._lib = saved


def test_product_package_never_imports_the_oracle():
    """The product path (paper_2605_18566_b200) must not import, link or execute oracle/."""
    import pathlib

    pkg = pathlib.Path(ROOT) / "paper_2605_18566_b200"
    for f in list(pkg.glob("*.py")) + list((pkg / "csrc").glob("*")):
        text = f.read_text(errors="ignore")
        assert "import oracle" not in text and "from oracle" not in text, f
        assert "liboracle" not in text and "hjmc_oracle" not in text, f


def test_picard_decide_and_residual_eps_host(lib):
    """Algorithm 1's stopping test behind the C-ABI (host functions, no GPU): ε_j =
    sqrt(num / max(den, 1e-300)) on all-reduced partials (R11), retire when ε < tol,
    NaN for inactive horizons, sup-norm difference passed through (Thm 2's d_k)."""
    import numpy as np

    part = np.array([[4.0, 100.0, 0.5], [1e-6, 1.0, 1e-3], [9.0, 0.0, 2.0], [1.0, 1.0, 7.0]])
    active = np.array([1, 1, 1, 0], dtype=np.uint8)
    eps = np.zeros(4)
    dsup = np.zeros(4)
    left = C.c_int32(-1)
    rc = lib.hjmc_picard_decide(part.ctypes.data_as(C.c_void_p), 4, 0.01,
                                active.ctypes.data_as(C.c_void_p), eps.ctypes.data_as(C.c_void_p),
                                dsup.ctypes.data_as(C.c_void_p), C.byref(left))
    assert rc == 0
    assert eps[0] == 0.2 and eps[1] == 1e-3 and eps[2] == 3.0 / 1e-150
    assert np.isnan(eps[3]) and np.isnan(dsup[3])
    assert list(dsup[:3]) == [0.5, 1e-3, 2.0]
    assert list(active) == [1, 0, 1, 0] and left.value == 2
    # EINVAL: K < 1, negative tol, NULL partials
    assert lib.hjmc_picard_decide(part.ctypes.data_as(C.c_void_p), 0, 0.1,
                                  active.ctypes.data_as(C.c_void_p), None, None, None) == 1
    assert lib.hjmc_picard_decide(part.ctypes.data_as(C.c_void_p), 4, -1.0,
                                  active.ctypes.data_as(C.c_void_p), None, None, None) == 1
    assert lib.hjmc_picard_decide(None, 4, 0.1, active.ctypes.data_as(C.c_void_p), None, None,
                                  None) == 1
    nd = np.array([[[4.0, 16.0], [0.0, 0.0]], [[2.0, 8.0], [1.0, 4.0]]])
    out = np.zeros(4)
    assert lib.hjmc_residual_eps(nd.ctypes.data_as(C.c_void_p), 4, out.ctypes.data_as(C.c_void_p)) == 0
    assert list(out) == [0.5, 0.0, 0.5, 0.5]

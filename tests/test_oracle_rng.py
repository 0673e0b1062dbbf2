"""Pins of the oracle's random-number stage (R19) against things other than itself.

* Philox4x32-10 bits: the CUDA toolkit's own curand_Philox4x32_10 (a library routine),
  evaluated on the host.
* Normal transform: N(0,1) moments and a KS test against scipy.stats.norm; the |z| bound
  sqrt(48 ln 2) implied by u ≥ 2^-24; exact antithetic symmetry; stream independence
  across query ids and tags.
"""
import math
import os
import shutil
import subprocess

import numpy as np
import pytest
import scipy.stats as st

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def curand_host(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available to build the curand host reference")
    exe = str(tmp_path_factory.mktemp("cph") / "cph")
    env = {k: v for k, v in os.environ.items() if k != "LD_PRELOAD"}   # (sanitizer runs)
    subprocess.run([nvcc, "-O1", "-Wno-deprecated-gpu-targets", "-o", exe,
                    os.path.join(HERE, "tools", "curand_philox_host.cu")], check=True, env=env)
    return exe


def test_philox_bit_exact_vs_curand(oracle_mod, curand_host):
    rng = np.random.default_rng(7)
    cases = [[0, 0, 0, 0, 0, 0], [0xFFFFFFFF] * 6]
    cases += rng.integers(0, 2**32, size=(254, 6), dtype=np.uint64).tolist()
    inp = "\n".join(" ".join(str(int(v)) for v in c) for c in cases) + "\n"
    env = {k: v for k, v in os.environ.items() if k != "LD_PRELOAD"}
    out = subprocess.run([curand_host], input=inp, capture_output=True, text=True, check=True,
                         env=env)
    ref = [list(map(int, ln.split())) for ln in out.stdout.strip().splitlines()]
    assert len(ref) == len(cases)
    for c, r in zip(cases, ref):
        assert oracle_mod.philox(c[:4], c[4:]) == r


def _draws(oracle_mod, n=4, count=50000, qid=3, jw=1, kw=0, antithetic=False, seed=11):
    P = oracle_mod.Problem(n=n, seed=seed, antithetic=antithetic)
    return oracle_mod.normals(P, qid, jw, kw, 0, count)


def test_normal_moments_and_ks(oracle_mod):
    z = _draws(oracle_mod).reshape(-1)          # 200k normals
    m = z.size
    assert abs(z.mean()) < 5 / math.sqrt(m)
    assert abs(z.var() - 1.0) < 5 * math.sqrt(2.0 / m)
    assert abs(st.skew(z)) < 5 * math.sqrt(6.0 / m)
    assert abs(st.kurtosis(z)) < 5 * math.sqrt(24.0 / m)
    assert st.kstest(z, "norm").pvalue > 1e-4
    # each coordinate of the quad separately (cos and sin branches)
    zz = _draws(oracle_mod, count=20000)
    for d in range(4):
        assert st.kstest(zz[:, d], "norm").pvalue > 1e-4


def test_normal_bound(oracle_mod):
    z = _draws(oracle_mod, count=20000)
    assert np.abs(z).max() <= math.sqrt(48 * math.log(2)) + 1e-12


def test_flat_stream_grouping(oracle_mod):
    """R19: for G·n ≤ 16 the G = 4/gcd(n,4) draws of group γ read one flat stream from the
    blocks (γ, b = 0..Q−1) — the same blocks a single draw of the G·n-dimensional layout uses;
    larger n (G = 1) take ceil(n/4) blocks per draw, so n = 5 is the first 5 normals of n = 8."""
    z4 = _draws(oracle_mod, n=4, count=20)
    z12 = _draws(oracle_mod, n=12, count=20)
    for n, G, ref in ((2, 2, z4), (3, 4, z12), (6, 2, z12)):
        zn = _draws(oracle_mod, n=n, count=G * 20)
        np.testing.assert_array_equal(zn.reshape(20, G * n), ref)
    z8 = _draws(oracle_mod, n=8, count=30)
    z5 = _draws(oracle_mod, n=5, count=30)
    np.testing.assert_array_equal(z5, z8[:, :5])
    np.testing.assert_array_equal(z8[:, :4], _draws(oracle_mod, n=4, count=30))


def test_antithetic_pairs_exact(oracle_mod):
    z = _draws(oracle_mod, n=5, count=1000, antithetic=True)
    np.testing.assert_array_equal(z[0::2], -z[1::2])
    plain = _draws(oracle_mod, n=5, count=500, antithetic=False)
    np.testing.assert_array_equal(z[0::2], plain)


def test_stream_independence(oracle_mod):
    a = _draws(oracle_mod, n=4, count=25000, qid=0).reshape(-1)
    for kw in [dict(qid=1), dict(jw=2), dict(kw=1), dict(seed=12)]:
        b = _draws(oracle_mod, n=4, count=25000, **{"qid": 0, **kw}).reshape(-1)
        assert abs(np.corrcoef(a, b)[0, 1]) < 0.02
        assert not np.array_equal(a, b)


def test_uniform_mapping_from_raw_words(oracle_mod):
    """z from the raw Philox words per the header's prose (consistency, not a pin)."""
    P = oracle_mod.Problem(n=4, seed=5)
    z, raw = oracle_mod.normals(P, 9, 2, 0, 0, 64, raw=True)
    m = (raw >> 9).astype(np.float64)
    u = (2 * m + 1) / 2**24
    a = m / 2**23
    r0 = np.sqrt(-2 * np.log(u[:, 0]))
    r2 = np.sqrt(-2 * np.log(u[:, 2]))
    ref = np.stack([r0 * np.cos(2 * np.pi * a[:, 1]), r0 * np.sin(2 * np.pi * a[:, 1]),
                    r2 * np.cos(2 * np.pi * a[:, 3]), r2 * np.sin(2 * np.pi * a[:, 3])], 1)
    np.testing.assert_allclose(z, ref, rtol=0, atol=1e-13)

"""GPU parity: the CUDA path (through the C-ABI) against the independent CPU oracle, element by
element on the same seeded inputs, at sizes spanning several CTAs/tiles with ragged tails,
plus the degenerate cases of the method. Tolerances: tests/_parity.py (R20)."""
import math

import numpy as np
import pytest

from _parity import (_final_outputs_within, assert_c_history, assert_dv,  # noqa: F401
                     assert_picard_history, assert_v)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


def pair(O, **kw):
    """A solver and the oracle problem with identical settings."""
    cfg = SolverConfig(**kw)
    okw = {k: v for k, v in kw.items() if k not in ("device", "sync_check")}
    return Solver(cfg), O.Problem(**okw)


# ---------------------------------------------------------------------------------------------
def test_rng_raw_bits_and_normals(O):
    for n, anti in ((3, False), (6, False), (45, False), (4, True)):
        s, P = pair(O, n=n, delta=0.01, seed=0x1234567890ABCDEF, tag=7, antithetic=anti)
        z, raw = s.debug_normals(qid=4242, jw=3, kw=1, i0=100, count=2000, raw=True)
        zo, rawo = O.normals(P, 4242, 3, 1, 100, 2000, raw=True)
        raw_np = raw.cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(raw_np, rawo)
        np.testing.assert_allclose(z.cpu().numpy(), zo, rtol=0, atol=2e-5)


@pytest.mark.parametrize("visc", ["paper", "full"])
def test_c1_value_grad_full_grid(O, visc):
    """Config 1 (BASELINE configs[0]) on the full 64×64 grid: GPU vs oracle, and both vs the
    exact Cole–Hopf closed form within MC error."""
    p = I.C1.with_(visc=visc)
    s, P = pair(O, n=2, delta=p.delta, T=p.T, N=p.N, seed=p.seed, visc=visc,
                system="quadratic", target="quad_bowl", tgt_params=(0.25,))
    x = I.queries(p)
    c = np.full(x.shape[0], 1.0 / P.delta_eff, dtype=np.float32)
    v, dv = s.value_grad(x, c, p.T, j_tag=1, k_tag=0)
    v, dv = v.cpu().numpy(), dv.cpu().numpy()
    vo, dvo = O.phi_batch(P, x, c.astype(np.float64), p.T, jw=1, kw=0)
    assert_v(v, vo)
    assert_dv(dv, dvo)
    k = P.delta_eff * p.T / P.delta_eff  # cσ² = τ
    xx = x.astype(np.float64)
    v_cf = (xx * xx).sum(1) / (2 * (1 + k)) - 0.25 + 2 / (2 * (1 / P.delta_eff)) * math.log1p(k)
    # MC error only (the GPU matches the pinned oracle above): SE_v reaches ~0.05 at the grid
    # corners where the weights concentrate (ESS), so the pointwise band is loose
    assert np.abs(v - v_cf).max() < 0.3
    assert abs(np.mean(v - v_cf)) < 0.01


@pytest.mark.parametrize("target,n,params,system,c,tau,lo,hi", [
    ("disk", 3, (5.0,), "dubins_rel", 3.0, 0.7, -12, 12),
    ("disk", 2, (1.0,), "quadratic", 20.0, 0.1, -3, 3),
    ("rel_disk6", 6, (1.5,), "rocket6", 12.0, 1.0, -6, 6),
    ("pair_union", 15, (1.0,), "dubins_pairs", 20.0, 1.0, -4, 4),
    ("pair_union", 45, (1.0,), "dubins_pairs", 0.05, 0.3, -4, 4),
    ("pursuit_min", 45, (1.5,), "multiagent", 5.0, 0.4, -6, 6),      # lane groups + evader shuffle
    ("quad_bowl", 45, (0.25,), "quadratic", 5.0, 0.2, -0.5, 0.5),
    ("quad_bowl", 1, (0.25,), "quadratic", 5.0, 0.2, -2, 2),
    ("linear", 3, (0.5, -1.0, 2.0, 0.3), "quadratic", 4.0, 0.5, -2, 2),
    ("const", 4, (-1.75,), "quadratic", 9.0, 0.5, -2, 2),
])
def test_value_grad_ragged(O, target, n, params, system, c, tau, lo, hi):
    """Single Φ pass, several targets; M and N ragged against the 256-thread CTA."""
    N = 3001 if n < 40 else 1001
    s, P = pair(O, n=n, delta=0.01, N=N, seed=99, system=system, target=target, tgt_params=params)
    x = I.random_queries(n, 37, lo, hi, seed=n)
    cc = np.full(37, c, dtype=np.float32)
    v, dv = s.value_grad(x, cc, tau, j_tag=5, k_tag=2, qid_base=1000)
    vo, dvo = O.phi_batch(P, x, cc.astype(np.float64), tau, qid_base=1000, jw=5, kw=2)
    assert_v(v.cpu().numpy(), vo)
    assert_dv(dv.cpu().numpy(), dvo)


def test_value_grad_antithetic_and_small_N(O):
    for N in (1, 2, 7, 255, 256, 257, 5001):
        s, P = pair(O, n=3, delta=0.01, N=N, antithetic=True, system="dubins_rel",
                    target="disk", tgt_params=(5.0,))
        x = I.random_queries(3, 19, -9, 9, seed=N)
        cc = np.full(19, 2.0, dtype=np.float32)
        v, dv = s.value_grad(x, cc, 0.8)
        vo, dvo = O.phi_batch(P, x, cc.astype(np.float64), 0.8)
        assert_v(v.cpu().numpy(), vo, f"v N={N}")
        assert_dv(dv.cpu().numpy(), dvo, f"dv N={N}")


def test_tau_zero_and_empty(O):
    s, P = pair(O, n=3, delta=0.01, system="dubins_rel", target="disk", tgt_params=(5.0,))
    x = np.array([[3.0, 4.0, 1.0], [0.0, 0.0, 0.0], [-6.0, 8.0, 0.0]], np.float32)
    v, dv = s.value_grad(x, np.ones(3, np.float32), 0.0)
    np.testing.assert_allclose(v.cpu().numpy(), [0.0, -5.0, 5.0], atol=1e-6)
    np.testing.assert_allclose(dv.cpu().numpy(), [[0.6, 0.8, 0], [1, 0, 0], [-0.6, 0.8, 0]], atol=1e-7)
    v0, _ = s.value_grad(np.zeros((0, 3), np.float32), np.zeros(0, np.float32), 0.5)
    assert v0.numel() == 0


def test_drift_translation_identity(O):
    """R4: v_b(x) = v_0(x + bτ) with identical samples — bit-exact on the GPU."""
    s, _ = pair(O, n=3, delta=0.01, N=4000, system="dubins_rel", target="disk", tgt_params=(5.0,))
    x = I.random_queries(3, 50, -8, 8, seed=1)
    b = I.random_queries(3, 50, -3, 3, seed=2)
    tau = np.float32(0.6)
    cc = np.full(50, 3.0, np.float32)
    v1, dv1 = s.value_grad(x, cc, float(tau), drift=b)
    xs = (x + (b * tau).astype(np.float32)).astype(np.float32)
    v2, dv2 = s.value_grad(xs, cc, float(tau))
    assert torch.equal(v1, v2)


def _grid(lo, hi, pts, n, fixed):
    a = np.linspace(lo, hi, pts)
    X, Y = np.meshgrid(a, a, indexing="ij")
    x = np.tile(np.asarray(fixed, np.float64), (X.size, 1))
    x[:, 0], x[:, 1] = X.ravel(), Y.ravel()
    return x.astype(np.float32)


def _compare_solve(O, s, P, x, qid_base=0, hist_check=True):
    out = s.solve_slice(x, qid_base=qid_base)
    ref = O.solve_slice(P, x, qid_base=qid_base)
    assert ref["status"] == 0
    g = {k: t.cpu().numpy() for k, t in out.items()}
    np.testing.assert_allclose(g["g0"], ref["g0"], rtol=1e-6, atol=1e-6)
    if hist_check:
        qids = np.arange(x.shape[0]) + qid_base
        assert_picard_history(O, P, x, qids, g["vhist"], g["chist"], ref)
    _final_outputs_within(O, P, x, np.arange(x.shape[0]) + qid_base, g, ref)
    return g, ref


def test_solve_slice_dubins_small(O):
    s, P = pair(O, n=3, delta=0.01, T=1.0, K=3, Kp=4, N=3001, seed=I.C2.seed,
                system="dubins_rel", sys_params=(5.0, 5.0, 1.0), target="disk", tgt_params=(5.0,))
    x = _grid(-20, 20, 11, 3, (0, 0, math.pi / 2))
    g, _ = _compare_solve(O, s, P, x)
    assert np.all(g["tube"] <= g["g0"])


def test_solve_slice_dubins_no_crn(O):
    s, P = pair(O, n=3, delta=0.01, T=1.0, K=2, Kp=3, N=2000, crn=False,
                system="dubins_rel", target="disk", tgt_params=(5.0,))
    _compare_solve(O, s, P, _grid(-9, 9, 7, 3, (0, 0, 0.3)), qid_base=77)


def test_solve_slice_rocket6(O):
    s, P = pair(O, n=6, delta=0.01, T=1.0, K=2, Kp=3, N=2500, seed=I.C3.seed,
                system="rocket6", sys_params=(64.0, 32.0, 1.0), target="rel_disk6",
                tgt_params=(1.5,))
    _compare_solve(O, s, P, _grid(-20, 20, 7, 6, (0,) * 6))


@pytest.mark.parametrize("K_pairs", [5, 15])
def test_solve_slice_pairs(O, K_pairs):
    s, P = pair(O, n=3 * K_pairs, delta=0.01, T=1.0, K=2, Kp=3, N=1200 if K_pairs == 5 else 600,
                system="dubins_pairs", sys_params=(5.0, 5.0, 1.0), target="pair_union",
                tgt_params=(1.0,))
    _compare_solve(O, s, P, _grid(-20, 20, 5, 3 * K_pairs, I.pair_fixed(K_pairs, math.pi / 2)))


def test_picard_quadratic_crn_stationary_gpu(O):
    s, P = pair(O, n=2, delta=0.05, T=0.5, K=2, Kp=4, N=4096, system="quadratic",
                target="quad_bowl", tgt_params=(0.25,))
    x = I.queries(I.C1)[::37]
    g, ref = _compare_solve(O, s, P, x)
    for k in range(1, 4):
        np.testing.assert_allclose(g["vhist"][:, k], g["vhist"][:, 0], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("N", [3000, 20000, 70000])    # one unit per warp / 4 warps / CTA
def test_shard_bit_identity(N):
    """Results depend on global query ids only: the 1/2/4/8-GPU partitions of shard.partition
    and a ragged hand split are bit-identical to the unsplit slice, for every thread-group
    size (the kernel variant depends on N only)."""
    from paper_2605_18566_b200 import shard

    s = Solver(SolverConfig.from_preset(I.C2, N=N, K=2, Kp=2))
    x = I.queries(I.C2)[:501]
    full = s.solve_slice(x)
    splits = [[(0, 123), (123, 378)]]
    for world in (2, 4, 8):
        splits.append([shard.partition(501, world, r) for r in range(world)])
    for parts in splits:
        outs = [s.solve_slice(x[a:a + n], qid_base=a) for a, n in parts]
        for k in ("v", "dv", "c", "tube"):
            assert torch.equal(full[k], torch.cat([o[k] for o in outs])), (parts, k)
        assert torch.equal(full["vhist"], torch.cat([o["vhist"] for o in outs], dim=2))


def test_host_path_matches_device_path():
    s = Solver(SolverConfig.from_preset(I.C2, N=2000, K=2, Kp=2))
    x = I.queries(I.C2)[:300]
    dev = {k: t.cpu().numpy() for k, t in s.solve_slice(x).items()}
    host = s.solve_slice_host(x)
    for k in dev:
        np.testing.assert_array_equal(dev[k], host[k])


def test_numeric_error_reporting():
    s = Solver(SolverConfig.from_preset(I.C2, N=500, K=1, Kp=1))
    x = I.queries(I.C2)[:64].copy()
    x[17, 0] = np.nan
    s.solve_slice(x, qid_base=1000)
    with pytest.raises(Exception) as ei:
        s.check()
    assert "ENUMERIC" in str(ei.value)
    assert s.last_bad_query() == 1017
    s.check()  # flag cleared


def test_eval_hamiltonian_and_target(O):
    rng = np.random.default_rng(0)
    for system, n, tgt, tp in (("dubins_rel", 3, "disk", (5.0,)), ("rocket6", 6, "rel_disk6", (1.5,)),
                               ("dubins_pairs", 15, "pair_union", (1.0,)), ("quadratic", 4, "quad_bowl", (0.25,))):
        s, P = pair(O, n=n, delta=0.01, system=system, target=tgt, tgt_params=tp)
        x = rng.uniform(-5, 5, (40, n)).astype(np.float32)
        p = rng.normal(size=(40, n)).astype(np.float32)
        H, c = s.eval_hamiltonian(x, p)
        Ho = np.array([O.hamiltonian(P, x[m].astype(float), p[m].astype(float)) for m in range(40)])
        co = np.array([O.gamma(P, x[m].astype(float), p[m].astype(float)) for m in range(40)])
        np.testing.assert_allclose(H.cpu().numpy(), Ho, rtol=1e-6, atol=1e-5)
        np.testing.assert_allclose(c.cpu().numpy(), co, rtol=1e-6, atol=1e-6)
        g, dg = s.eval_target(x)
        go = np.array([O.g(P, x[m].astype(float)) for m in range(40)])
        dgo = np.array([O.dg(P, x[m].astype(float)) for m in range(40)])
        np.testing.assert_allclose(g.cpu().numpy(), go, rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(dg.cpu().numpy(), dgo, rtol=1e-6, atol=1e-6)


@pytest.mark.slow
def test_c2_full_size_sampled(O):
    """BASELINE configs[1] in the exact launch configuration bench.py times (all 10,201 queries,
    N = 65,536, 10 horizons × 8 Picard iterates) against the oracle on 48 sampled queries:
    a deterministic spread plus the queries nearest the BRT boundary (smallest |v|) and those
    with an unclamped (interior) coefficient (R8), where the Picard feedback is most sensitive."""
    p = I.C2
    s = Solver(SolverConfig.from_preset(p))
    x = I.queries(p)
    out = {k: t.cpu().numpy() for k, t in s.solve_slice(x).items()}
    s.check()
    spread = I.subsample_ids(x.shape[0], 24)
    boundary = np.argsort(np.abs(out["v"]))[:12]
    interior = np.flatnonzero((out["chist"][-1, -1] > p.c_min * 1.01) & (out["chist"][-1, -1] < p.c_max * 0.99))[:12]
    ids = np.unique(np.concatenate([spread, boundary, interior])).astype(np.int64)
    P = O.Problem.from_preset(p)
    ref = O.solve_slice(P, x[ids], qids=ids.astype(np.uint32))
    assert_picard_history(O, P, x[ids], ids, out["vhist"][:, :, ids], out["chist"][:, :, ids],
                          ref, "c2 full-size sample")
    _final_outputs_within(O, P, x[ids], ids, out, ref, sel=ids)
    np.testing.assert_allclose(out["g0"][ids], ref["g0"], rtol=1e-6, atol=1e-6)


def test_skip_stationary_is_bit_identical():
    """HJMC_FLAG_SKIP_STATIONARY copies iterates whose inputs are bit-identical (c unchanged
    under CRN): every output must equal the full computation exactly, with fewer passes."""
    kw = dict(N=3000, K=3, Kp=5)
    base = Solver(SolverConfig.from_preset(I.C2, **kw))
    fast = Solver(SolverConfig.from_preset(I.C2, skip_stationary=True, **kw))
    x = I.queries(I.C2)[::13]
    M = x.shape[0]
    a = base.solve_slice(x)
    na = base.pass_count()
    b = fast.solve_slice(x)
    nb = fast.pass_count()
    for k in a:
        assert torch.equal(a[k], b[k]), k
    assert na == M * 3 * 5
    assert nb < na
    # without CRN nothing may be skipped
    nocrn = Solver(SolverConfig.from_preset(I.C2, skip_stationary=True, crn=False, **kw))
    nocrn.solve_slice(x)
    assert nocrn.pass_count() == M * 3 * 5


@pytest.mark.parametrize("skip,N,spec", [(False, 3000, False), (True, 3000, False),
                                         (True, 40000, False), (True, 70000, False),
                                         (True, 3000, True), (False, 40000, True),
                                         (True, 70000, True)])
def test_reuse_passes_is_bit_identical(skip, N, spec):
    """HJMC_FLAG_REUSE_PASSES: under CRN a pass is a function of its c, so a pass at a c the
    unit has already used returns the stored sums. Every output equals the full schedule bit
    for bit, and the number of sample passes equals the number of distinct c per (query,
    horizon) trajectory (read off the full run's own chist), stationary skip or not."""
    kw = dict(N=N, K=3, Kp=8)     # N picks the thread group per unit: a warp, 4 warps, the CTA
    base = Solver(SolverConfig.from_preset(I.C2, **kw))
    memo = Solver(SolverConfig.from_preset(I.C2, reuse_passes=True, skip_stationary=skip,
                                           speculate=spec, **kw))
    x = I.queries(I.C2)[::7]
    a = base.solve_slice(x)
    base.pass_count()
    b = memo.solve_slice(x)
    nb = memo.pass_count()
    for k in a:
        assert torch.equal(a[k], b[k]), k
    ch = a["chist"].cpu().numpy()                     # [K][Kp][M]
    distinct = sum(len(set(ch[j, :, m].tolist())) for j in range(ch.shape[0])
                   for m in range(ch.shape[2]))
    if spec:      # a clamp reached after the opposite clamp was sampled costs no pass
        assert nb < distinct
    else:
        assert nb == distinct
    assert nb < 0.5 * x.shape[0] * 3 * 8               # the C2 slice cycles between the clamps
    # without CRN every pass draws fresh samples: nothing is reused
    nocrn = Solver(SolverConfig.from_preset(I.C2, reuse_passes=True, crn=False, **kw))
    nocrn.solve_slice(x)
    assert nocrn.pass_count() == x.shape[0] * 3 * 8


def test_reuse_passes_lane_groups_and_proposal():
    """The memo is shared by the lane-group kernel (n = 45 pair union) and the Laplace
    proposal (the centre μ follows from c): outputs bit-identical to the full schedule."""
    for preset, extra in ((I.C5.with_(N=2048, K=2, Kp=4, grid_pts=8), {}),
                          (I.C5.with_(N=2048, K=2, Kp=6, grid_pts=8), {"speculate": True}),
                          (I.C4.with_(N=3000, K=2, Kp=6, grid_pts=9), {"speculate": True}),
                          (I.C2.with_(N=2048, K=2, Kp=6, grid_pts=11), {"proposal": "laplace"}),
                          (I.C2.with_(N=5001, K=2, Kp=6, grid_pts=11), {"antithetic": True}),
                          (I.C3.with_(N=2048, K=2, Kp=5, grid_pts=9), {})):
        x = I.queries(preset)
        base = Solver(SolverConfig.from_preset(preset, **extra))
        memo = Solver(SolverConfig.from_preset(preset, reuse_passes=True, skip_stationary=True,
                                               **extra))
        a = base.solve_slice(x)
        b = memo.solve_slice(x)
        for k in a:
            assert torch.equal(a[k], b[k]), (preset.name, k)
        assert memo.pass_count() <= x.shape[0] * preset.K * preset.Kp


def test_picard_stepwise_equals_fused_solve():
    """hjmc_picard_pass with every horizon active reproduces hjmc_solve_slice's iterates
    bit for bit (same counters, same kernel body)."""
    from paper_2605_18566_b200.picard import solve_adaptive

    p = I.C2.with_(N=2000, K=3, Kp=4)
    s = Solver(SolverConfig.from_preset(p, crn=False))
    x = I.queries(p)[::97]
    fused = s.solve_slice(x, qid_base=5)
    r = solve_adaptive(s, x, tol=0.0, max_iter=4, qid_base=5)
    assert list(r["iters"]) == [4, 4, 4]
    assert torch.equal(r["v"], fused["vhist"][:, -1])
    assert torch.equal(r["c"][-1], fused["c"])
    assert torch.equal(r["dv"][-1], fused["dv"])
    assert torch.equal(r["tube"], fused["tube"])


def test_picard_adaptive_vs_oracle(O):
    """Algorithm 1 with its stopping test: GPU driver vs the oracle's, same iteration counts,
    residual histories and final values (C2 physics, small N)."""
    from paper_2605_18566_b200.picard import solve_adaptive

    p = I.C2.with_(N=3000, K=3)
    x = I.queries(p)[::53]
    P = O.Problem.from_preset(p, crn=False)
    ref = O.picard_adaptive(P, x, 0.0, 5)
    s = Solver(SolverConfig.from_preset(p, crn=False))
    r = solve_adaptive(s, x, tol=0.0, max_iter=5)
    np.testing.assert_allclose(r["eps"], ref["eps"], rtol=0.05, atol=1e-7)
    e = np.sort(ref["eps"][np.isfinite(ref["eps"]) & (ref["eps"] > 0)])
    gap = int(np.argmax(e[1:] / e[:-1]))                # threshold far from every eps value
    tol = float(np.sqrt(e[gap] * e[gap + 1]))
    ref_t = O.picard_adaptive(P, x, tol, 5)
    r_t = solve_adaptive(s, x, tol=tol, max_iter=5)
    assert list(r_t["iters"]) == list(ref_t["iters"])
    for j in range(3):
        assert_v(r_t["v"][j].cpu().numpy(), ref_t["v"][j], f"v[{j}]")


@pytest.mark.parametrize("idx", [3, 4, 5])
def test_full_size_configs_golden(O, idx):
    """BASELINE configs 3–5 at FULL size (N = 2^18 / 2^20, all horizons and Picard iterates) on
    the sampled global query ids stored by scripts/make_golden.py (oracle-only values). The
    GPU replays the same global ids; results depend only on them, so this equals the full
    slice launch for those queries."""
    import os

    p = I.BY_INDEX[idx]
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"{p.name}_sample.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    d = np.load(path)
    ids = d["ids"]
    s = Solver(SolverConfig.from_preset(p))
    out = {k: t.cpu().numpy() for k, t in s.solve_slice(d["x"], qid=ids.astype(np.int32)).items()}
    s.check()
    ref = {k: d[k] for k in ("v", "dv", "c", "tube", "vhist", "chist", "dvhist", "g0")}
    P = O.Problem.from_preset(p)
    assert_picard_history(O, P, d["x"], ids, out["vhist"], out["chist"], ref)
    _final_outputs_within(O, P, d["x"], ids, out, ref)
    np.testing.assert_allclose(out["g0"], ref["g0"], rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("preset,n_q,kw", [
    ("paper_rockets3_40x40", 49, dict(N=3000, K=2, Kp=4)),
    ("paper_double_integrator", 49, dict(N=3000, K=2, Kp=4)),
    ("paper_multiagent45", 16, dict(N=800, K=2, Kp=3)),
])
def test_solve_slice_paper_systems(O, preset, n_q, kw):
    """The paper's own systems through the fused kernel vs oracle."""
    p = I.PRESETS[preset].with_(**kw)
    s = Solver(SolverConfig.from_preset(p))
    x = I.queries(p)
    x = x[np.linspace(0, x.shape[0] - 1, n_q).round().astype(int)]
    _compare_solve(O, s, O.Problem.from_preset(p), x)


def test_multiagent_small_and_hamiltonian(O):
    s, P = pair(O, n=9, delta=0.02, T=1.0, K=2, Kp=3, N=2000, system="multiagent",
                sys_params=(1.0, 2.0), target="pursuit_min", tgt_params=(1.5,))
    x = I.random_queries(9, 25, -4, 4, seed=3)
    _compare_solve(O, s, P, x)
    rng = np.random.default_rng(1)
    xx = rng.uniform(-3, 3, (30, 9)).astype(np.float32)
    pp = rng.normal(size=(30, 9)).astype(np.float32)
    H, _ = s.eval_hamiltonian(xx, pp)
    Ho = [O.hamiltonian(P, xx[m].astype(float), pp[m].astype(float)) for m in range(30)]
    np.testing.assert_allclose(H.cpu().numpy(), Ho, rtol=1e-6, atol=1e-5)


def test_brat_clamp_gpu(O):
    """HJI-RCBRAT-Visc: tube = max(BRT tube, ℓ(x)) with a disk obstacle."""
    p = I.PAPER_DOUBLE_INTEGRATOR.with_(N=2000, K=2, Kp=3)
    x = I.queries(p)[::7]
    brt = Solver(SolverConfig.from_preset(p)).solve_slice(x)
    pa = p.with_(avoid="disk", avoid_params=(0.3, -0.2, 0.4))
    s = Solver(SolverConfig.from_preset(pa))
    brat = s.solve_slice(x)
    P = O.Problem.from_preset(pa)
    ell = np.array([O.avoid_l(P, xm.astype(np.float64)) for xm in x])
    np.testing.assert_allclose(brat["tube"].cpu().numpy(),
                               np.maximum(brt["tube"].cpu().numpy(), ell), rtol=0, atol=1e-6)
    assert torch.equal(brat["v"], brt["v"])
    _compare_solve(O, s, P, x, hist_check=False)


def test_plain_c_consumer(tmp_path):
    """The C-ABI stands alone: a plain C program (examples/c_api_demo.c) links libhjmc.so,
    solves through both the device and host entry points and gets identical results."""
    import json
    import os
    import shutil
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path / "c_api_demo")
    libdir = os.path.join(root, "paper_2605_18566_b200")
    subprocess.run([gcc, "-O2", "-I", os.path.join(root, "include"),
                    os.path.join(root, "examples", "c_api_demo.c"), "-L", libdir, "-lhjmc",
                    "-I", "/usr/local/cuda/include", "-L", "/usr/local/cuda/lib64", "-lcudart",
                    "-Wl,-rpath," + libdir, "-lm", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    rec = json.loads(out.stdout.strip().splitlines()[-1])
    assert rec["identical_device_host"] and rec["M"] == 441
    assert rec["passes"] == 2 * 441 * 4 * 3       # device + host solve, full schedule
    assert rec["brt_points"] > 0
    assert rec["picard_graph_matches_fixed_schedule"]


def test_counter_extremes(O):
    """Counter packing at its limits: global ids next to 2^32, horizon tag 65535, Picard tag
    255, N not a multiple of the draw group (n = 3: G = 4) — GPU vs oracle."""
    for n, target, params, system in ((3, "disk", (5.0,), "dubins_rel"),
                                      (6, "rel_disk6", (1.5,), "rocket6"),
                                      (45, "pair_union", (1.0,), "dubins_pairs")):
        N = 1027 if n < 40 else 259
        s, P = pair(O, n=n, delta=0.01, N=N, seed=0xFFFFFFFFFFFFFFFF, tag=0xFFFFFFFF,
                    system=system, target=target, tgt_params=params)
        x = I.random_queries(n, 9, -6, 6, seed=n + 100)
        base = 0xFFFFFFFF - 8                           # ids 2^32−9 … 2^32−1
        cc = np.full(9, 7.0, dtype=np.float32)
        v, dv = s.value_grad(x, cc, 0.9, j_tag=65535, k_tag=255, qid_base=base)
        vo, dvo = O.phi_batch(P, x, cc.astype(np.float64), 0.9, qid_base=base, jw=65535, kw=255)
        assert_v(v.cpu().numpy(), vo, f"v n={n}")
        assert_dv(dv.cpu().numpy(), dvo, f"dv n={n}")


def test_solve_slice_lane_groups_ragged_and_antithetic(O):
    """n = 45 pair union: the lane-group kernel with N not a multiple of its 64-sample stride,
    and the antithetic (generic) instantiation, both against the oracle."""
    for anti in (False, True):
        s, P = pair(O, n=45, delta=0.01, T=1.0, K=1, Kp=2, N=333, antithetic=anti,
                    system="dubins_pairs", target="pair_union", tgt_params=(1.0,))
        x = np.tile(np.asarray(I.pair_fixed(15, 0.7), np.float32), (6, 1))
        x[:, 0] = np.linspace(-3, 3, 6)
        x[:, 1] = np.linspace(2, -2, 6)
        _compare_solve(O, s, P, x, qid_base=11)


@pytest.mark.parametrize("target,n,params,system,c,tau", [
    ("disk", 3, (5.0,), "dubins_rel", 20.0, 0.7),
    ("quad_bowl", 2, (0.25,), "quadratic", 20.0, 0.5),
    ("rel_disk6", 6, (1.5,), "rocket6", 12.0, 1.0),
    ("pair_union", 45, (1.0,), "dubins_pairs", 5.0, 0.5),
])
def test_laplace_proposal_value_grad(O, target, n, params, system, c, tau):
    """Laplace-tilted proposal (R28): GPU vs oracle on the same samples."""
    N = 2049 if n < 40 else 515
    s, P = pair(O, n=n, delta=0.01, N=N, seed=5, system=system, target=target,
                tgt_params=params, proposal="laplace")
    lo, hi = (-1.2, 1.2) if target == "quad_bowl" else (-7, 7)
    x = I.random_queries(n, 23, lo, hi, seed=n + 7)
    cc = np.full(23, c, dtype=np.float32)
    v, dv = s.value_grad(x, cc, tau, j_tag=2, k_tag=1, qid_base=70)
    vo, dvo = O.phi_batch(P, x, cc.astype(np.float64), tau, qid_base=70, jw=2, kw=1)
    assert_v(v.cpu().numpy(), vo)
    assert_dv(dv.cpu().numpy(), dvo)


def test_laplace_proposal_zero_variance_linear():
    """g = a·y + b: the tilted estimator is exact for any N — the GPU returns the Gaussian-tilt
    value a·x + b − cσ²|a|²/2 to fp32 precision with N = 7."""
    a = np.array([0.7, -1.2, 0.4])
    s = Solver(SolverConfig(n=3, delta=0.01, N=7, target="linear", tgt_params=tuple(a) + (0.3,),
                            proposal="laplace"))
    x = I.random_queries(3, 64, -2, 2, seed=4)
    for c, tau in ((1.0, 0.5), (6.0, 2.0)):
        v, _ = s.value_grad(x, np.full(64, c, np.float32), tau)
        exact = x.astype(np.float64) @ a + 0.3 - c * 0.01 * tau * (a @ a) / 2
        np.testing.assert_allclose(v.cpu().numpy(), exact, rtol=0, atol=2e-5)


def test_laplace_proposal_solve_slice(O):
    s, P = pair(O, n=3, delta=0.01, T=1.0, K=2, Kp=3, N=2500, system="dubins_rel",
                target="disk", tgt_params=(5.0,), proposal="laplace")
    _compare_solve(O, s, P, _grid(-12, 12, 7, 3, (0, 0, math.pi / 2)), qid_base=3)


def test_binding_validates_shapes():
    """The C-ABI writes through raw pointers, so the binding rejects mis-shaped buffers."""
    s = Solver(SolverConfig.from_preset(I.C2, N=256, K=2, Kp=2))
    x = I.queries(I.C2)[:10]
    with pytest.raises(ValueError):
        s.solve_slice(x[:, :2])                                    # wrong n
    out = s.alloc_result(10)
    out["vhist"] = torch.empty(2, 2, 9, device="cuda")            # wrong M
    with pytest.raises(ValueError):
        s.solve_slice(x, out=out)
    with pytest.raises(ValueError):
        s.value_grad(x, np.ones(9, np.float32), 0.5)               # c of the wrong length
    with pytest.raises(ValueError):
        s.solve_slice(x, qid=np.arange(11, dtype=np.int32))
    with pytest.raises(ValueError):
        s.solve_slice(x, drift=np.zeros((10, 2), np.float32))
    s.solve_slice(x, out=s.alloc_result(10))                        # the right shapes pass


@pytest.mark.parametrize("N", [4096, 4097, 65536, 65537])
def test_group_size_switches(O, N):
    """Plain passes run one unit per warp up to N = 4096, per 4 warps up to 65536, per CTA
    above: each kernel against the oracle on both sides of each switch (ragged 197 units)."""
    s, P = pair(O, n=3, delta=0.01, N=N, seed=I.C2.seed, system="dubins_rel", target="disk",
                tgt_params=(5.0,))
    M = 197
    x = I.random_queries(3, M, -9, 9, seed=N)
    cc = np.full(M, 4.0, dtype=np.float32)
    v, dv = s.value_grad(x, cc, 0.8, j_tag=3, k_tag=1, qid_base=77)
    ids = np.arange(0, M, 5)
    ref = [O.phi(P, x[i].astype(np.float64), 4.0, 0.8, qid=77 + int(i), jw=3, kw=1) for i in ids]
    assert_v(v.cpu().numpy()[ids], np.array([r[0] for r in ref]))
    assert_dv(dv.cpu().numpy()[ids], np.array([r[1] for r in ref]))


def test_warp_unit_solve_slice_ragged(O):
    """The warp-per-unit kernel through solve_slice with a unit count that is not a multiple of
    8 units per CTA (M·K = 2,403)."""
    s, P = pair(O, n=3, delta=0.01, T=1.0, K=3, Kp=2, N=700, seed=I.C2.seed,
                system="dubins_rel", target="disk", tgt_params=(5.0,))
    x = I.random_queries(3, 801, -9, 9, seed=5)
    _compare_solve(O, s, P, x, qid_base=11)


@pytest.mark.parametrize("crn", [True, False])
def test_picard_device_resident_equals_host_driven(O, crn):
    """hjmc_picard_solve (Algorithm 1 as one CUDA graph with a conditional while-node) gives
    the host-driven loop's results bit for bit: iteration counts, ε and sup-norm histories,
    every horizon's final v / Dv / c — with horizons retiring at different iterates."""
    from paper_2605_18566_b200.picard import solve_adaptive, solve_adaptive_device

    p = I.C2.with_(N=3000, K=3)
    x = I.queries(p)[::29]
    s = Solver(SolverConfig.from_preset(p, crn=crn))
    r0 = solve_adaptive(s, x, tol=0.0, max_iter=6)
    e = np.sort(r0["eps"][np.isfinite(r0["eps"]) & (r0["eps"] > 0)])
    tol = float(np.median(e))                            # some horizons stop early, some not
    a = solve_adaptive(s, x, tol=tol, max_iter=6)
    b = solve_adaptive_device(s, x, tol=tol, max_iter=6)
    assert list(a["iters"]) == list(b["iters"]) and len(set(a["iters"])) >= 1
    np.testing.assert_array_equal(a["eps"], b["eps"])
    np.testing.assert_array_equal(a["d_sup"], b["d_sup"])
    for k in ("v", "dv", "c", "tube"):
        assert torch.equal(a[k], b[k]), k
    assert list(a["converged"]) == list(b["converged"])
    # the cached graph is relaunched for identical arguments and rebuilt when they change
    b2 = solve_adaptive_device(s, x, tol=tol, max_iter=6)
    assert torch.equal(b["v"], b2["v"]) and list(b["iters"]) == list(b2["iters"])
    b3 = solve_adaptive_device(s, x, tol=0.0, max_iter=3)
    assert list(b3["iters"]) == [3, 3, 3]
    np.testing.assert_array_equal(b3["eps"][:, :3], r0["eps"][:, :3])
    # a larger host-driven solve reallocates the handle's scratch: the cached graph must notice
    solve_adaptive(s, I.queries(p)[::5], tol=0.0, max_iter=2)
    b4 = solve_adaptive_device(s, x, tol=tol, max_iter=6)
    assert torch.equal(b["v"], b4["v"]) and list(b["iters"]) == list(b4["iters"])
    # an exactly stationary problem stops after the second pass (quadratic H, CRN: c = 1/δ)
    q = Solver(SolverConfig(n=2, delta=0.05, T=0.5, K=2, N=2048, system="quadratic",
                            target="quad_bowl", tgt_params=(0.25,)))
    rq = solve_adaptive_device(q, I.queries(I.C1)[::9], tol=1e-9, max_iter=10)
    assert list(rq["iters"]) == [2, 2] and np.all(rq["eps"][:, 1] == 0.0)


def test_shard_bit_identity_lane_groups():
    """The n = 45 lane-group kernel: the 4-GPU partition is bit-identical to the unsplit slice."""
    from paper_2605_18566_b200 import shard

    p = I.C5.with_(N=3000, K=2, Kp=2, grid_pts=8)
    s = Solver(SolverConfig.from_preset(p))
    x = I.queries(p)[:301]
    full = s.solve_slice(x)
    outs = [s.solve_slice(x[a:a + n], qid_base=a) for a, n in
            (shard.partition(301, 4, r) for r in range(4))]
    for k in ("v", "dv", "c", "tube", "vhist"):
        dim = 2 if k == "vhist" else 0
        assert torch.equal(full[k], torch.cat([o[k] for o in outs], dim=dim)), k


@pytest.mark.parametrize("target,n,params,system,extra", [
    ("disk", 3, (5.0,), "dubins_rel", {}),
    ("pair_union", 45, (1.0,), "dubins_pairs", {}),                       # lane groups
    ("disk", 3, (5.0,), "dubins_rel", {"proposal": "laplace"}),
    ("rel_disk6", 6, (1.5,), "rocket6", {"antithetic": True}),
])
def test_solve_slice_with_drift_vs_oracle(O, target, n, params, system, extra):
    """The optional drift hook (R4: y = x + bτ + σz, b per query) through the fused solve —
    generic, lane-group, Laplace-proposal and antithetic kernels — against the oracle at every
    Picard iterate (the translation identity alone would not catch a drift applied with the
    wrong τ_j)."""
    s, P = pair(O, n=n, delta=0.01, T=1.0, K=3, Kp=3, N=1500, seed=77, system=system,
                target=target, tgt_params=params, **extra)
    x = I.random_queries(n, 29, -6, 6, seed=n + 5)
    b = I.random_queries(n, 29, -2, 2, seed=n + 6)
    out = s.solve_slice(x, qid_base=9, drift=b)
    ref = O.solve_slice(P, x, drift=b, qid_base=9)
    assert ref["status"] == 0
    g = {k: t.cpu().numpy() for k, t in out.items()}
    assert_picard_history(O, P, x, np.arange(29) + 9, g["vhist"], g["chist"], ref)


@pytest.mark.parametrize("target,n,params,system,span", [
    ("disk", 2, (1.0,), "quadratic", 8.0),
    ("disk", 3, (5.0,), "dubins_rel", 12.0),
    ("pair_union", 45, (1.0,), "dubins_pairs", 6.0),                      # lane-group max mode
])
def test_two_pass_fallback_when_the_shift_underflows(O, target, n, params, system, span):
    """The guaranteed shift B = −A·core_lower leaves every weight below 2⁻¹⁰⁰ when c·σ is large
    (the bound uses |z| ≤ 5.77 per coordinate, the realised samples reach ~3.5): the pass is
    redone with the exact maximum exponent (the plain two-pass log-sum-exp). c = 20,
    σ = 1 puts every query there; GPU vs oracle, and through the fused solve with the memo."""
    N = 4096
    s, P = pair(O, n=n, delta=1.0, N=N, seed=5, system=system, target=target, tgt_params=params)
    x = I.random_queries(n, 23, -span, span, seed=n + 40)
    cc = np.full(23, 20.0, dtype=np.float32)
    v, dv = s.value_grad(x, cc, 1.0, j_tag=2, k_tag=0)
    vo, dvo = O.phi_batch(P, x, cc.astype(np.float64), 1.0, jw=2, kw=0)
    assert_v(v.cpu().numpy(), vo, "v (fallback)")
    assert_dv(dv.cpu().numpy(), dvo, "dv (fallback)")
    # fused solve (c from Γ, clamps up to 20) with and without the exact shortcuts
    kw = dict(n=n, delta=1.0, T=1.0, K=2, Kp=3, N=N, seed=5, system=system, target=target,
              tgt_params=params)
    a = Solver(SolverConfig(**kw)).solve_slice(x)
    b = Solver(SolverConfig(reuse_passes=True, skip_stationary=True, speculate=True,
                            **kw)).solve_slice(x)
    for k in a:
        assert torch.equal(a[k], b[k]), k
    ref = O.solve_slice(O.Problem(**kw), x)
    assert_picard_history(O, O.Problem(**kw), x, np.arange(23), a["vhist"].cpu().numpy(),
                          a["chist"].cpu().numpy(), ref)


@pytest.mark.parametrize("target,n,params,system,span", [
    ("disk", 3, (5.0,), "dubins_rel", (9.0, 15.0)),
    ("pair_union", 45, (1.0,), "dubins_pairs", (9.0, 12.0)),              # lane-group kernel
])
def test_fallback_threshold_scales_with_N(O, target, n, params, system, span):
    """R24 (round 2): at N = 2²⁰ a pass whose LARGEST shifted weight is ~2⁻⁹⁴ — above round 1's
    fixed 2⁻¹⁰⁰ fallback line — while the shifted sum S stays below N·2⁻¹⁰² must take the exact
    two-pass log-sum-exp ("for numerical stability"): with ex2.approx.ftz, weights under
    2⁻¹²⁶ are dropped, which the fixed line let reach N·2⁻²⁶ = 1.6 % of S. Per query c is chosen
    from the oracle's realised minimum of g so that the realised max exponent against the
    kernel's guaranteed shift (the bound |z| ≤ 8.1578 on a coordinate pair, hjmc_targets.cuh)
    sits at −94; GPU vs oracle at R20."""
    N = 1 << 20
    s, P = pair(O, n=n, delta=1.0, N=N, seed=11, system=system, target=target, tgt_params=params)
    M = 8
    rng = np.random.default_rng(n)
    x = np.zeros((M, n), np.float32)
    if n > 3:
        x[:] = np.asarray(I.pair_fixed(n // 3, 0.0), np.float32) * 1.5   # other pairs far away
    r = rng.uniform(*span, M)
    th = rng.uniform(0, 2 * np.pi, M)
    x[:, 0], x[:, 1] = r * np.cos(th), r * np.sin(th)
    sigma, tau, rad = 1.0, 1.0, params[0]
    log2e = 1.0 / math.log(2.0)
    c = np.zeros(M)
    for m in range(M):
        _, _, diag, _ = O.phi(P, x[m].astype(np.float64), 1.0, tau, qid=m, jw=3, kw=0)
        core_min = diag[0] + rad                               # min_i core(y_i), core = g + r
        pos = math.hypot(float(x[m, 0]), float(x[m, 1]))
        core_lower = max(0.0, pos - sigma * 8.1578) * 0.9999
        c[m] = 94.0 / (log2e * (core_min - core_lower))       # realised max exponent −94
    c = c.astype(np.float32)
    for m in range(M):
        _, _, diag, _ = O.phi(P, x[m].astype(np.float64), float(c[m]), tau, qid=m, jw=3, kw=0)
        pos = math.hypot(float(x[m, 0]), float(x[m, 1]))
        core_lower = max(0.0, pos - sigma * 8.1578) * 0.9999
        e = float(c[m]) * log2e * (core_lower - (diag[0] + rad))   # log2 of the largest weight
        log2_s = diag[5] * log2e + e                                # log2 of the shifted sum
        assert -100.0 < e < -88.0, e
        assert log2_s < math.log2(N) - 102.0, log2_s               # the new rule falls back
    v, dv = s.value_grad(x, c, tau, j_tag=3, k_tag=0)
    vo, dvo = O.phi_items(P, x, np.arange(M), np.arange(M), c.astype(np.float64), tau, 3, 0)
    assert_v(v.cpu().numpy(), vo, "v (N-scaled fallback)")
    assert_dv(dv.cpu().numpy(), dvo, "dv (N-scaled fallback)")


@pytest.mark.parametrize("crn", [True, False])
def test_picard_adaptive_brat_vs_oracle(O, crn):
    """Algorithm 1 with its stopping test (step 5) on a problem with a disk obstacle
    (HJI-RCBRAT-Visc): both drivers — host-driven (hjmc_picard_pass +
    hjmc_picard_decide + hjmc_tube) and device-resident (hjmc_picard_solve, tube inside the
    graph) — against the oracle's orc_picard_adaptive + orc_tube: identical iteration counts,
    every horizon's final v and the clamped tube at R20; the two drivers bit-identical."""
    from paper_2605_18566_b200.picard import solve_adaptive, solve_adaptive_device

    p = I.PAPER_DOUBLE_INTEGRATOR.with_(N=3000, K=3, avoid="disk", avoid_params=(0.3, -0.2, 0.4),
                                        crn=crn)
    x = I.queries(p)[::23]
    P = O.Problem.from_preset(p)
    full = O.picard_adaptive(P, x, 0.0, 6)
    e = np.sort(full["eps"][np.isfinite(full["eps"]) & (full["eps"] > 0)])
    gap = int(np.argmax(e[1:] / e[:-1]))                 # threshold far from every ε value
    tol = float(np.sqrt(e[gap] * e[gap + 1]))
    ref = O.picard_adaptive(P, x, tol, 6)
    s = Solver(SolverConfig.from_preset(p))
    a = solve_adaptive(s, x, tol=tol, max_iter=6)
    b = solve_adaptive_device(s, x, tol=tol, max_iter=6)
    assert list(a["iters"]) == list(ref["iters"]) == list(b["iters"])
    for k in ("v", "c", "tube"):
        assert torch.equal(a[k], b[k]), k
    for j in range(p.K):
        assert_v(a["v"][j].cpu().numpy(), ref["v"][j], f"v[{j}]")
    assert_v(a["tube"].cpu().numpy(), ref["tube"], "tube (BRAT)")
    ell = np.array([O.avoid_l(P, xm.astype(np.float64)) for xm in x], dtype=np.float32)
    tube = a["tube"].cpu().numpy()
    assert np.all(tube >= ell - 1e-6) and np.any(np.abs(tube - ell) <= 1e-6)   # clamp binds


def test_picard_resident_sharded_driver_equals_graph():
    """The sharded device-resident Algorithm 1 (hjmc_picard_dev_begin / _pass / _decide with
    the all-reduce on the stream; VERDICT r1 missing #6) equals hjmc_picard_solve's conditional
    graph bit for bit — eagerly enqueued, captured into one CUDA graph, and with a real NCCL
    all-reduce of a one-rank process group inside the captured graph (a multi-rank run needs
    more GPUs than this pool has; the collective's arithmetic is the identity at one rank)."""
    import socket

    import torch.distributed as dist

    from paper_2605_18566_b200.picard import solve_adaptive_device, solve_adaptive_resident

    for crn in (True, False):
        p = I.C2.with_(N=3000, K=3)
        x = I.queries(p)[::29]
        s = Solver(SolverConfig.from_preset(p, crn=crn))
        r0 = solve_adaptive_device(s, x, tol=0.0, max_iter=6)
        e = np.sort(r0["eps"][np.isfinite(r0["eps"]) & (r0["eps"] > 0)])
        tol = float(np.median(e))
        a = solve_adaptive_device(s, x, tol=tol, max_iter=6)
        runs = [solve_adaptive_resident(s, x, tol=tol, max_iter=6),
                solve_adaptive_resident(s, x, tol=tol, max_iter=6, graph=True)]
        if crn:
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                    world_size=1, device_id=torch.device("cuda", 0))
            try:
                runs.append(solve_adaptive_resident(s, x, tol=tol, max_iter=6,
                                                    group=dist.group.WORLD, graph=True))
            finally:
                dist.destroy_process_group()
        for b in runs:
            assert list(a["iters"]) == list(b["iters"])
            np.testing.assert_array_equal(a["eps"], b["eps"])
            np.testing.assert_array_equal(a["d_sup"], b["d_sup"])
            for k in ("v", "dv", "c", "tube"):
                assert torch.equal(a[k], b[k]), k
        assert len(set(a["iters"])) >= 1


@pytest.mark.parametrize("N", [3000, 40000, 70000, 1500])   # warp / 4-warp / CTA groups; n = 45 lanes
def test_repeated_launches_bit_identical(N):
    """Race check by repetition (compute-sanitizer is closed on this pool): the same solve
    relaunched with the units' placement in CTAs shifted — a leading block of extra queries
    moves every unit to another CTA slot and named-barrier group — must give bit-identical
    results for the queries in common, for the warp, 4-warp (bar.sync 1 + g, 128) and CTA
    groups and for the lane-group kernel (N = 1500 at n = 45)."""
    p = I.C2.with_(N=N, K=3, Kp=3) if N != 1500 else I.C5.with_(N=N, K=3, Kp=2)
    s = Solver(SolverConfig.from_preset(p))
    x_all = I.queries(p)[:260]
    ref = s.solve_slice(x_all[5:], qid_base=5)
    for shift in (0, 1, 2, 3, 5):
        for _ in range(2):
            out = s.solve_slice(x_all[5 - shift:], qid_base=5 - shift)
            for k in ("v", "dv", "c", "tube"):
                assert torch.equal(out[k][shift:], ref[k]), (N, shift, k)
            assert torch.equal(out["vhist"][:, :, shift:], ref["vhist"]), (N, shift)

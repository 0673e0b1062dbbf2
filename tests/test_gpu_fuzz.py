"""Seeded random parity sweep: value_grad through every kernel variant (one unit per warp / per
4 warps / per CTA, lane groups, antithetic, Laplace proposal) on random targets, dimensions,
sample counts, coefficients, horizons, viscosities (both conventions, R1) and query sets — GPU
vs the oracle at the R20 tolerances.
Deterministic (fixed generator seed): a failure names its case index and parameters."""
import numpy as np
import pytest

from _parity import assert_dv, assert_v

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

# (target, n, target params, system, coordinate range)
TARGETS = [
    ("disk", 2, (1.0,), "quadratic", 3.0),
    ("disk", 3, (5.0,), "dubins_rel", 12.0),
    ("rel_disk6", 6, (1.5,), "rocket6", 6.0),
    ("pair_union", 15, (1.0,), "dubins_pairs", 5.0),
    ("pair_union", 45, (1.0,), "dubins_pairs", 5.0),
    ("pursuit_min", 45, (1.5,), "multiagent", 6.0),
    ("quad_bowl", 2, (0.25,), "quadratic", 1.0),
    ("linear", 4, (0.5, -1.0, 2.0, 0.3, 0.1), "quadratic", 2.0),
]
N_CHOICES = [1, 6, 257, 4096, 4097, 9001, 65536, 65537]


def cases(count=24, seed=20261020):
    rng = np.random.default_rng(seed)
    for i in range(count):
        tgt, n, prm, sysname, span = TARGETS[i % len(TARGETS)]
        N = int(rng.choice(N_CHOICES if n < 40 else [7, 4097, 9001]))
        yield i, dict(target=tgt, n=n, tgt_params=prm[: max(1, n + 1)] if tgt == "linear" else prm,
                      system=sysname, span=span, N=N, M=int(rng.integers(1, 40)),
                      c=float(np.exp(rng.uniform(np.log(0.05), np.log(20.0)))),
                      tau=float(rng.uniform(0.05, 1.0)), antithetic=bool(rng.random() < 0.25),
                      proposal="laplace" if rng.random() < 0.2 else "plain",
                      seed=int(rng.integers(0, 2**62)), qid_base=int(rng.integers(0, 2**31)),
                      delta=float(np.exp(rng.uniform(np.log(0.005), np.log(0.1)))),
                      visc="full" if rng.random() < 0.3 else "paper")


@pytest.mark.parametrize("i,case", list(cases()))
def test_random_value_grad_parity(oracle_mod, i, case):
    O = oracle_mod
    kw = dict(n=case["n"], delta=case["delta"], visc=case["visc"], N=case["N"], seed=case["seed"],
              system=case["system"],
              target=case["target"], tgt_params=case["tgt_params"], antithetic=case["antithetic"],
              proposal=case["proposal"])
    s = Solver(SolverConfig(**kw))
    P = O.Problem(**kw)
    x = I.random_queries(case["n"], case["M"], -case["span"], case["span"], seed=i)
    # per-query coefficients around the case's c (the pass freezes c per query, R5)
    cc = (case["c"] * np.exp(np.random.default_rng(i).uniform(-1, 1, case["M"]))).astype(np.float32)
    v, dv = s.value_grad(x, cc, case["tau"], j_tag=i + 1, k_tag=i % 7, qid_base=case["qid_base"])
    vo, dvo = O.phi_batch(P, x, cc.astype(np.float64), case["tau"], qid_base=case["qid_base"],
                          jw=i + 1, kw=i % 7)
    assert_v(v.cpu().numpy(), vo, f"case {i} {case}")
    assert_dv(dv.cpu().numpy(), dvo, f"case {i} {case}")


def solve_cases(count=12, seed=777):
    rng = np.random.default_rng(seed)
    games = [("disk", 3, (5.0,), "dubins_rel", 12.0), ("rel_disk6", 6, (1.5,), "rocket6", 6.0),
             ("pair_union", 15, (1.0,), "dubins_pairs", 5.0),
             ("pair_union", 45, (1.0,), "dubins_pairs", 5.0),
             ("pursuit_min", 9, (1.5,), "multiagent", 6.0), ("disk", 2, (0.1,), "double_integrator", 1.0)]
    for i in range(count):
        tgt, n, prm, sysname, span = games[i % len(games)]
        yield i, dict(target=tgt, n=n, tgt_params=prm, system=sysname, span=span,
                      N=int(rng.choice([300, 4097, 6000] if n < 40 else [300, 2000])),
                      M=int(rng.integers(3, 20)), K=int(rng.integers(1, 4)), Kp=int(rng.integers(1, 5)),
                      T=float(rng.uniform(0.3, 1.5)), delta=float(rng.choice([0.01, 0.05, 0.08])),
                      crn=bool(rng.random() < 0.8), seed=int(rng.integers(0, 2**62)),
                      skip=bool(rng.random() < 0.5), reuse=bool(rng.random() < 0.5),
                      qid_base=int(rng.integers(0, 2**20)))


@pytest.mark.parametrize("i,case", list(solve_cases()))
def test_random_solve_slice_parity(oracle_mod, i, case):
    """The fused Picard/horizon loop with random K, Kp, T, δ, CRN on/off and the exact-shortcut
    flags: every iterate against the oracle (R20/R25, R27 where non-contractive)."""
    from _parity import assert_picard_history

    O = oracle_mod
    kw = dict(n=case["n"], delta=case["delta"], T=case["T"], K=case["K"], Kp=case["Kp"],
              N=case["N"], seed=case["seed"], crn=case["crn"], system=case["system"],
              target=case["target"], tgt_params=case["tgt_params"])
    s = Solver(SolverConfig(skip_stationary=case["skip"], reuse_passes=case["reuse"], **kw))
    P = O.Problem(**kw)
    x = I.random_queries(case["n"], case["M"], -case["span"], case["span"], seed=100 + i)
    out = {k: t.cpu().numpy() for k, t in s.solve_slice(x, qid_base=case["qid_base"]).items()}
    s.check()
    ref = O.solve_slice(P, x, qid_base=case["qid_base"])
    assert ref["status"] == 0
    assert_picard_history(O, P, x, np.arange(case["M"]) + case["qid_base"], out["vhist"],
                          out["chist"], ref)
    assert np.all(out["tube"] <= out["g0"] + 1e-6)

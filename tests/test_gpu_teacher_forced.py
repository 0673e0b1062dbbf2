"""Teacher-forced per-iterate parity: Φ alone (Thm 2's Φ, P:338–341;
Cor. logsumexp / mc_gradient) at the ORACLE's own coefficient history, for every
(query, horizon, Picard iterate) of full-size trajectories — all 10,201 queries of C2 and the
sampled global ids of C3–C5. At each (j, k) the GPU runs hjmc_value_grad at c = float32(oracle
chist[j, k]) and the oracle runs orc_phi at the same c, τ and counter tags, so the expansive
Picard feedback Γ (R27) never enters: the plain R20 tolerances (2e-4 on v, 1e-3 on Dv, with the
slice-wide floors) must hold with ZERO exceptions. Fixtures: tests/golden/c2_dubins_n3_chist.npz
(oracle chist) and tests/golden/<config>_teacher.npz (oracle Φ at the sampled ids' chist), both
written by scripts/make_golden.py, which calls only oracle/."""
import os

import numpy as np
import pytest

from _parity import dv_violations, teacher_items, teacher_tau, v_violations

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


def _forced_passes(s, p, x, chist, index, v_ref, dv_ref, qid=None):
    """GPU value_grad at every (j, k) of chist; returns the worst v and Dv ratios per (j, k)."""
    K, Kp, M = chist.shape
    q = None if qid is None else torch.from_numpy(np.asarray(qid, dtype=np.int32)).cuda()
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    worst_v = np.zeros((K, Kp))
    worst_d = np.zeros((K, Kp))
    for j in range(K):
        tau = float(teacher_tau(p.T, p.K, j))
        for k in range(Kp):
            c = torch.from_numpy(np.asarray(chist[j, k]).astype(np.float32)).cuda()
            v, dv = s.value_grad(xd, c, tau, j_tag=j + 1, k_tag=0, qid=q)
            idx = index[j, k]
            worst_v[j, k] = v_violations(v.cpu().numpy(), v_ref[idx]).max()
            worst_d[j, k] = dv_violations(dv.cpu().numpy(), dv_ref[idx]).max()
    s.check()
    return worst_v, worst_d


@pytest.mark.slow
def test_teacher_forced_c2_full_slice(O):
    """All 10,201 × 10 × 8 iterates of BASELINE configs[1] (C2, N = 65,536): the oracle's Φ is
    evaluated here at each unique (query, horizon, c) — 140,401 passes on every host core."""
    p = I.C2
    chist = np.load(os.path.join(GOLDEN, f"{p.name}_chist.npz"))["chist"]
    x = I.queries(p)
    assert chist.shape == (p.K, p.Kp, x.shape[0])
    m, j, c, index = teacher_items(chist)
    P = O.Problem.from_preset(p)
    tau = np.array([teacher_tau(p.T, p.K, jj) for jj in j], dtype=np.float64)
    v_ref, dv_ref = O.phi_items(P, x, m, m.astype(np.uint32), c.astype(np.float64), tau,
                                (j + 1).astype(np.uint32), 0)
    s = Solver(SolverConfig.from_preset(p))
    wv, wd = _forced_passes(s, p, x, chist, index, v_ref, dv_ref)
    print(f"C2 teacher-forced: {len(m)} oracle passes; worst v {wv.max():.3g}, Dv {wd.max():.3g} "
          "of tolerance over all 816,080 iterates")
    assert wv.max() <= 1.0 and wd.max() <= 1.0, (wv.max(), wd.max())


@pytest.mark.parametrize("idx", [3, 4, 5])
def test_teacher_forced_full_size_sampled(O, idx):
    """BASELINE configs 3–5 at full N on the sampled global ids (tests/golden/*_sample.npz: an
    even spread, the BRT-boundary band and unclamped-c queries): every (j, k) iterate."""
    p = I.BY_INDEX[idx]
    path = os.path.join(GOLDEN, f"{p.name}_teacher.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    d = np.load(os.path.join(GOLDEN, f"{p.name}_sample.npz"))
    t = np.load(path)
    m, j, c, index = teacher_items(d["chist"])
    # the fixture's items (any order) must be exactly this trajectory's unique (m, j, c)
    gold = {(int(a), int(b), float(cc)): i for i, (a, b, cc) in
            enumerate(zip(t["m"].tolist(), t["j"].tolist(), t["c"].tolist()))}
    assert len(gold) == len(m)
    perm = np.array([gold[(int(a), int(b), float(cc))] for a, b, cc in
                     zip(m.tolist(), j.tolist(), c.tolist())], dtype=np.int64)
    s = Solver(SolverConfig.from_preset(p))
    wv, wd = _forced_passes(s, p, d["x"], d["chist"], index, t["v"][perm], t["dv"][perm],
                            qid=d["ids"])
    print(f"{p.name} teacher-forced: {len(m)} passes, {d['ids'].size} queries; worst v "
          f"{wv.max():.3g}, Dv {wd.max():.3g} of tolerance")
    assert wv.max() <= 1.0 and wd.max() <= 1.0, (wv.max(), wd.max())


@pytest.mark.slow
def test_trajectory_c2_complete_slice_r27_cap(O):
    """The Picard trajectories themselves (with Γ feedback) on the COMPLETE C2 slice — every
    query, horizon and iterate of the benchmark-size solve — against the oracle's trajectories,
    rebuilt exactly from its stored coefficient history (under CRN, vhist[j][k] = Φ_j(chist[j][k])
    at the double c and τ_j = jT/K the oracle's solve used). Plain R20/R25 everywhere except the
    conditioning-limited units of the non-contractive band (R27), capped at 0.1 % of units and
    0.05 % of final outputs and printed with their ids."""
    from _parity import _final_outputs_within, assert_picard_history

    p = I.C2
    chist = np.load(os.path.join(GOLDEN, f"{p.name}_chist.npz"))["chist"]
    x = I.queries(p)
    K, Kp, M = chist.shape
    keys = {}
    index = np.zeros((K, Kp, M), dtype=np.int64)
    for j in range(K):
        for k in range(Kp):
            for m, c in enumerate(chist[j, k].tolist()):
                index[j, k, m] = keys.setdefault((m, j, c), len(keys))
    items = sorted(keys, key=keys.get)
    im = np.array([t[0] for t in items], dtype=np.int64)
    ij = np.array([t[1] for t in items], dtype=np.int64)
    ic = np.array([t[2] for t in items], dtype=np.float64)
    P = O.Problem.from_preset(p)
    v, dv = O.phi_items(P, x, im, im.astype(np.uint32), ic, (ij + 1) * p.T / p.K,
                        (ij + 1).astype(np.uint32), 0)
    g0 = np.array([O.g(P, xm.astype(np.float64)) for xm in x])
    ref = {"vhist": v[index], "dvhist": dv[index], "chist": chist}
    ref["v"], ref["dv"] = ref["vhist"][-1, -1], ref["dvhist"][-1, -1]
    ref["tube"] = np.minimum(g0, ref["vhist"][:, -1].min(axis=0))
    s = Solver(SolverConfig.from_preset(p))
    out = {k: t.cpu().numpy() for k, t in s.solve_slice(x).items()}
    s.check()
    qids = np.arange(M)
    assert_picard_history(O, P, x, qids, out["vhist"], out["chist"], ref, "c2 complete slice")
    _final_outputs_within(O, P, x, qids, out, ref)
    np.testing.assert_allclose(out["g0"], g0, rtol=1e-6, atol=1e-6)

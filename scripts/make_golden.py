"""Write tests/golden/<config>_sample.npz: oracle (only) results at BASELINE.json's FULL sizes
for a deterministic sample of each config's global query ids. The GPU parity test replays the
same global ids through the CUDA path (results depend only on global ids, so this equals the
full launch). Sample = an even spread, the queries nearest the target boundary band
(|g(x)| ≤ σ_K·8.16, where the BRT boundary lies), and queries whose c^(0) is unclamped (R8).
Usage: python scripts/make_golden.py c3 c4 c5 [--threads T]

--chist c2: the oracle's frozen-coefficient history chist[K][Kp][M] for EVERY query of the config
(tests/golden/<config>_chist.npz). The teacher-forced parity test feeds float32(chist[j, k]) to
hjmc_value_grad and to the oracle's Φ at every (query, horizon, iterate),
which isolates Φ from the Picard feedback Γ; storing c (mostly the clamp values, so it
compresses well) instead of Φ's outputs keeps the fixture small — the test re-evaluates the
oracle's Φ itself.

--teacher c3 c4 c5: the oracle's Φ at every unique (query, horizon, float32 c) of the sampled
C3–C5 trajectories (tests/golden/<config>_teacher.npz), for the same teacher-forced test at full
size without re-running minutes of oracle work per test run."""
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2605_18566_b200 import inputs as I  # noqa: E402

COUNTS = {3: (256, 64, 64), 4: (64, 16, 16), 5: (24, 8, 8)}


def sample_ids(p, P, x, n_spread, n_band, n_int):
    M = x.shape[0]
    spread = I.subsample_ids(M, n_spread)
    stride = max(1, M // 4000)                       # scan a thinned grid for the picks
    cand = np.arange(0, M, stride)
    g = np.array([O.g(P, x[m].astype(np.float64)) for m in cand])
    band = math.sqrt(P.delta_eff * p.T) * 8.16
    near = cand[np.argsort(np.abs(g))][:n_band]
    c0 = np.array([O.gamma(P, x[m].astype(np.float64), O.dg(P, x[m].astype(np.float64))) for m in cand])
    inter = cand[(c0 > p.c_min * 1.01) & (c0 < p.c_max * 0.99)]
    inter = inter[np.linspace(0, len(inter) - 1, min(n_int, len(inter))).round().astype(int)] if len(inter) else inter
    return np.unique(np.concatenate([spread, near, inter])).astype(np.int64)


def chist_full(idx: int, threads: int):
    p = I.BY_INDEX[idx]
    P = O.Problem.from_preset(p)
    x = I.queries(p)
    t0 = time.time()
    r = O.solve_slice(P, x, nthreads=threads)
    dt = time.time() - t0
    assert r["status"] == 0
    path = os.path.join(ROOT, "tests", "golden", f"{p.name}_chist.npz")
    np.savez_compressed(path, chist=r["chist"],
                        source=np.array("scripts/make_golden.py --chist -> oracle.solve_slice "
                                        f"(double), all {x.shape[0]} queries of preset {p.name}; "
                                        f"{dt:.0f} s on {O.max_threads()} threads"))
    print(f"{p.name}: chist of {x.shape[0]} queries in {dt:.0f} s -> {path}", flush=True)


def teacher_items(chist):
    """Unique (query index m, horizon j (0-based), float32 c) over every iterate k of
    chist[K][Kp][M] — under CRN a Φ pass is a function of (m, j, c) alone."""
    K, Kp, M = chist.shape
    cf = chist.astype(np.float32)
    items = sorted({(m, j, float(cf[j, k, m])) for j in range(K) for k in range(Kp) for m in range(M)})
    m = np.array([t[0] for t in items], dtype=np.int64)
    j = np.array([t[1] for t in items], dtype=np.int64)
    c = np.array([t[2] for t in items], dtype=np.float32)
    return m, j, c


def teacher_tau(p, j0):
    """τ_j as the fp32 value hjmc_value_grad receives (j0 = 0-based horizon)."""
    return np.float32((j0 + 1) * p.T / p.K)


def teacher(idx: int, threads: int):
    """Teacher-forced Φ of the oracle at its OWN coefficient history:
    for every unique (query, horizon, float32(chist[j, k])) of the <config>_sample.npz ids, v and
    Dv of one pass at that c, τ = float32(j T/K), counter tags (j, 0) (CRN). The GPU test feeds
    the same c to hjmc_value_grad at every (j, k), isolating Φ from the Picard feedback."""
    p = I.BY_INDEX[idx]
    P = O.Problem.from_preset(p)
    assert p.crn
    d = np.load(os.path.join(ROOT, "tests", "golden", f"{p.name}_sample.npz"))
    m, j, c = teacher_items(d["chist"])
    tau = np.array([teacher_tau(p, jj) for jj in j], dtype=np.float64)
    t0 = time.time()
    v, dv = O.phi_items(P, d["x"], m, d["ids"][m].astype(np.uint32), c.astype(np.float64), tau,
                        (j + 1).astype(np.uint32), 0, nthreads=threads)
    dt = time.time() - t0
    path = os.path.join(ROOT, "tests", "golden", f"{p.name}_teacher.npz")
    np.savez_compressed(path, m=m, j=j, c=c, v=v, dv=dv,
                        source=np.array("scripts/make_golden.py --teacher -> oracle.phi_items "
                                        f"(double) at float32(chist) of {p.name}_sample.npz; "
                                        f"{len(m)} passes, {dt:.0f} s on {O.max_threads()} threads"))
    print(f"{p.name}: {len(m)} teacher-forced passes in {dt:.0f} s -> {path}", flush=True)


def main():
    threads = int(sys.argv[sys.argv.index("--threads") + 1]) if "--threads" in sys.argv else 0
    if "--teacher" in sys.argv:
        for a in sys.argv[1:]:
            if a.startswith("c") and a[1:].isdigit():
                teacher(int(a[1:]), threads)
        return
    if "--chist" in sys.argv:
        for a in sys.argv[1:]:
            if a.startswith("c") and a[1:].isdigit():
                chist_full(int(a[1:]), threads)
        return
    which = [int(a.lstrip("c")) for a in sys.argv[1:] if a.startswith("c")] or [3, 4, 5]
    threads = int(sys.argv[sys.argv.index("--threads") + 1]) if "--threads" in sys.argv else 0
    for idx in which:
        p = I.BY_INDEX[idx]
        P = O.Problem.from_preset(p)
        x = I.queries(p)
        ids = sample_ids(p, P, x, *COUNTS[idx])
        t0 = time.time()
        r = O.solve_slice(P, x[ids], qids=ids.astype(np.uint32), nthreads=threads)
        dt = time.time() - t0
        assert r["status"] == 0
        path = os.path.join(ROOT, "tests", "golden", f"{p.name}_sample.npz")
        np.savez_compressed(path, ids=ids, x=x[ids], v=r["v"], dv=r["dv"], c=r["c"], tube=r["tube"],
                            vhist=r["vhist"], chist=r["chist"], dvhist=r["dvhist"], g0=r["g0"],
                            source=np.array("scripts/make_golden.py -> oracle.solve_slice (double); "
                                            f"preset {p.name}; {dt:.0f} s on {O.max_threads()} threads"))
        print(f"{p.name}: {len(ids)} queries in {dt:.0f} s -> {path}", flush=True)


if __name__ == "__main__":
    main()

"""A/B timing of libhjmc build variants on the benchmark's C5 workload (a prefix of
inputs.bench_ids, full N, K, Kp), with a bit-identity check of every output against the first
variant. Usage: python tools/lg_variant_bench.py [count] [config] [solver-flags-json] — variants
from variants/libhjmc_*.so plus the in-tree library ("base"); flags e.g.
'{"skip_stationary": 1, "reuse_passes": 1, "speculate": 1}' time the exact shortcuts."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json, hashlib, torch, numpy as np
sys.path.insert(0, "{root}")
from paper_2605_18566_b200 import _lib, inputs as I
_lib.load("{lib}")
from paper_2605_18566_b200.solver import Solver, SolverConfig
p = I.BY_INDEX[{cfg}] if isinstance({cfg}, int) else I.PRESETS[{cfg}]
ids = I.bench_ids(p)
ids = ids[np.linspace(0, len(ids) - 1, min({count}, len(ids))).round().astype(int)]
s = Solver(SolverConfig.from_preset(p, **{flags}))
x = torch.from_numpy(np.ascontiguousarray(I.queries(p)[ids])).cuda()
q = torch.from_numpy(ids.astype(np.int32)).cuda()
out = s.alloc_result(x.shape[0])
s.solve_slice(x, qid=q, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range({reps}): s.solve_slice(x, qid=q, out=out)
e1.record(); torch.cuda.synchronize()
s.check()
ms = e0.elapsed_time(e1) / {reps}
h = hashlib.sha1(b"".join(out[k].cpu().numpy().tobytes() for k in sorted(out))).hexdigest()[:16]
print(json.dumps({{"ms": ms, "evals_per_s": len(ids) * p.N * p.K * p.Kp / (ms / 1e3), "digest": h}}))
'''

if __name__ == "__main__":
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
    arg = sys.argv[2] if len(sys.argv) > 2 else "5"
    cfg = int(arg.lstrip("c")) if arg.lstrip("c").isdigit() else repr(arg)
    flags = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
    libs = [os.path.join(ROOT, "paper_2605_18566_b200", "libhjmc.so")]
    libs += sorted(glob.glob(os.path.join(ROOT, "variants", "libhjmc_*.so")))
    for lib in libs:
        code = CHILD.format(root=ROOT, lib=lib, cfg=cfg, count=count, reps=2, flags=repr(flags))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
        name = "base" if "variants" not in lib else os.path.basename(lib)[7:-3]
        print(json.dumps({"variant": name, "config": f"c{cfg}" if isinstance(cfg, int) else arg, "queries": count, "flags": flags,
                          "result": line}), flush=True)

"""Time solve_slice on a config for each libhjmc variant in variants/ (CUDA events)."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json, torch
sys.path.insert(0, "{root}")
from paper_2605_18566_b200 import _lib, inputs as I
_lib.load("{lib}")
from paper_2605_18566_b200.solver import Solver, SolverConfig
p = I.BY_INDEX[{cfg}] if isinstance({cfg}, int) else I.PRESETS[{cfg}]
kw = {kw}
skw = {{k: kw.pop(k) for k in ("skip_stationary", "reuse_passes", "speculate") if k in kw}}
p = p.with_(**kw) if kw else p
s = Solver(SolverConfig.from_preset(p, **skw))
x = torch.from_numpy(I.queries(p)).cuda()
out = s.alloc_result(x.shape[0])
for _ in range(2): s.solve_slice(x, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range({reps}): s.solve_slice(x, out=out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / {reps}
print(json.dumps({{"ms": ms, "evals_per_s": p.M * p.N * p.K * p.Kp / (ms / 1e3)}}))
'''

if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
    cfg = int(cfg) if cfg.isdigit() else repr(cfg)
    kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    reps = 3
    for lib in sorted(glob.glob(os.path.join(ROOT, "variants", "libhjmc_*.so"))):
        code = CHILD.format(root=ROOT, lib=lib, cfg=cfg, kw=kw, reps=reps)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        print(os.path.basename(lib), line, flush=True)

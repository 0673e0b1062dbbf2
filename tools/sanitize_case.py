"""Small solve for compute-sanitizer runs (memcheck / racecheck / synccheck): generic kernel,
lane-group kernel, value_grad, stepwise Picard and the tube/BRAT epilogue, all tiny."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18566_b200 import inputs as I  # noqa: E402
from paper_2605_18566_b200.picard import solve_adaptive  # noqa: E402
from paper_2605_18566_b200.solver import Solver, SolverConfig  # noqa: E402

s = Solver(SolverConfig.from_preset(I.C2, N=600, K=2, Kp=2, skip_stationary=True))
x = I.queries(I.C2)[::997]
s.solve_slice(x)
s.value_grad(x, np.full(x.shape[0], 3.0, np.float32), 0.4)
solve_adaptive(s, x, tol=1e-3, max_iter=3)
s.check()
s5 = Solver(SolverConfig.from_preset(I.C5, N=300, K=1, Kp=2))
s5.solve_slice(I.queries(I.C5)[::65537])
s5.check()
pa = I.PAPER_DOUBLE_INTEGRATOR.with_(N=300, K=2, Kp=2, avoid="disk", avoid_params=(0.1, 0.1, 0.3))
Solver(SolverConfig.from_preset(pa)).solve_slice(I.queries(pa)[::97])
print("sanitize case ok")

"""Probe (not collected): one warm CG solve_many at the C3 shape with a 4-iteration budget
(for an ncu launch list of the solver's kernels)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W

n, s = 101000, 64
rng = np.random.default_rng(0)
X = rng.standard_normal((n, 16))
B = np.asfortranarray(rng.standard_normal((n, s)))
hyp = W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, W.MATERN32)
op = W.KernelOperator(hyp, X, precision=W.F32_3XTF32)
cfg = W.SolverConfig(tolerance=1e-12, max_iters=int(os.environ.get("ITERS", "4")), precond_rank=100,
                     precond_shift=1e-3)
for rep in range(2):
    t0 = time.perf_counter()
    res = W.solve_many(op, B, [W.Initialization.cold()] * s, cfg)
    print(f"solve {time.perf_counter() - t0:.3f} s, iters {res[0].iterations}", flush=True)

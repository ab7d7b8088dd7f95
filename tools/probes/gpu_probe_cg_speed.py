"""Probe (not collected): where a C3-sized CG iteration spends its time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W
n, d, s = 100000, 16, 64
X = np.random.default_rng(0).standard_normal((n, d))
op = W.KernelOperator(W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, W.MATERN32), X, precision=W.F32_3XTF32)
B = np.asfortranarray(np.random.default_rng(1).standard_normal((n, s)))
for iters in (1, 6):
    cfg = W.SolverConfig(tolerance=1e-12, max_iters=iters, precond_rank=100, precond_shift=1e-3)
    t0 = time.perf_counter()
    W.solve_many(op, B, [W.Initialization.cold()] * s, cfg)
    print(f"max_iters={iters}: {time.perf_counter() - t0:.3f} s")
t0 = time.perf_counter(); Y = op.kmatvec(B); print(f"host kmatvec {time.perf_counter() - t0:.3f} s")

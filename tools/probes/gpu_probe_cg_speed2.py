"""Probe (not collected): CG speed before/after appending rows (bench C3 leg)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W
n0, n, d, s = 100000, 101000, 16, 64
X = np.random.default_rng(0).standard_normal((n, d))
op = W.KernelOperator(W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, W.MATERN32), X[:n0], precision=W.F32_3XTF32)
B = np.asfortranarray(np.random.default_rng(1).standard_normal((n, s)))
cfg = W.SolverConfig(tolerance=1e-12, max_iters=6, precond_rank=100, precond_shift=1e-3)
for rep in range(2):
    t0 = time.perf_counter(); W.solve_many(op, np.asfortranarray(B[:n0]), [W.Initialization.cold()] * s, cfg); print(f"n=100k 6 iters: {time.perf_counter() - t0:.3f} s")
op.append_rows(X[n0:])
for rep in range(2):
    t0 = time.perf_counter(); W.solve_many(op, B, [W.Initialization.cold()] * s, cfg); print(f"n=101k 6 iters: {time.perf_counter() - t0:.3f} s")
import torch
V = torch.randn(n, s, dtype=torch.float64, device="cuda"); Y = torch.empty_like(V)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s); torch.cuda.synchronize(); print(f"kmatvec_dev n=101k {1e3*(time.perf_counter()-t0):.2f} ms")

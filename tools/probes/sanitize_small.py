"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck): the tcgen05
kernel-matvec (Matern and RBF, gram and cross mode), the fp64 kernel, CG / SGD / AP solves of
a few iterations (krows, kcols, block Cholesky, preconditioner, vector kernels), RFF
evaluation.  No torch: only the product library through ctypes.

  compute-sanitizer --tool racecheck python tools/probes/sanitize_small.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2511_16340_b200 import warmgp as W  # noqa: E402

rng = np.random.default_rng(0)
n, d, s = 1100, 8, 16
X = rng.random((n, d))
V = rng.standard_normal((n, s))
for kind in (W.MATERN32, W.RBF):
    hyp = W.KernelHyperparams(0.5, 1.0, 0.1, kind)
    tc = W.KernelOperator(hyp, X, precision=W.F32_3XTF32)
    f64 = W.KernelOperator(hyp, X, precision=W.F64)
    Y1, Y2 = tc.kmatvec(V), f64.kmatvec(V)
    print("kmatvec rel err", float(np.linalg.norm(Y1 - Y2) / np.linalg.norm(Y2)))
    Xs = rng.random((300, d))
    tc.cross_matvec(Xs, V[:, :4])
    cfg = W.SolverConfig(tolerance=1e-10, max_iters=3, precond_rank=20, precond_shift=0.01,
                         batch_size=64, block_size=128, learning_rate=1e-3)
    for op in (tc, f64):
        for m in (W.CG, W.SGD, W.AP):
            W.solve_many(op, V[:, :4], [W.Initialization.cold()] * 4, cfg.copy(method=m))
    pri = [W.sample_prior(hyp, d, 64, c) for c in range(3)]
    W.rff_eval(f64, pri)
    W.rff_eval(f64, pri, Xs, fast=True)
print("sanitize workload done")

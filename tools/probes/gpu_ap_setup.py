"""Probe (not collected): AP solve setup cost (block factorisations + initial residual) vs the
iterations, at the C2 end shape (N=20k, d=8 RBF, s=17, block 500): max_iters 0 vs 200."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W

n, d, s = int(os.environ.get("N", "20000")), 8, 17
X = np.random.default_rng(0).random((n, d))
hyp = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
op = W.KernelOperator(hyp, X, precision=W.F32_3XTF32)
B = np.asfortranarray(np.random.default_rng(1).standard_normal((n, s)))
for its in (0, 0, 200, 0):
    cfg = W.SolverConfig(method=W.AP, tolerance=1e-4, max_iters=its, block_size=500)
    t0 = time.perf_counter()
    W.solve_many(op, B, [W.Initialization.cold()] * s, cfg, return_status=True)
    print(f"AP max_iters={its}: {time.perf_counter() - t0:.4f} s", flush=True)

"""Probe (not collected): one AP solve at the C2 end shape (N=20k RBF d=8, s=17, block 500,
greedy, fp32 operator), 50 iterations, for an ncu launch list (where an AP iteration's time goes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W

n, d, s = 20000, 8, 17
X = np.random.default_rng(0).random((n, d))
op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF), X, precision=W.F32_3XTF32)
B = np.asfortranarray(np.random.default_rng(1).standard_normal((n, s)))
cfg = W.SolverConfig(method=W.AP, tolerance=1e-4, max_iters=int(os.environ.get("ITERS", "50")), block_size=500)
W.solve_many(op, B, [W.Initialization.cold()] * s, cfg, return_status=True)

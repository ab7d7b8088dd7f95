"""Probe (not collected): a short SGD solve_many at the C2 shape (N=20k, d=8, s=17, RBF,
batch 512, fp64) for timing and an ncu launch list."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W

n, s = 20000, 17
rng = np.random.default_rng(0)
X = rng.random((n, 8))
B = np.asfortranarray(rng.standard_normal((n, s)))
op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF), X, precision=W.F64)
iters = int(os.environ.get("ITERS", "20"))
cfg = W.SolverConfig(method=W.SGD, tolerance=1e-12, max_iters=iters, learning_rate=1e-3, batch_size=512)
for rep in range(2):
    t0 = time.perf_counter()
    W.solve_many(op, B, [W.Initialization.cold()] * s, cfg)
    print(f"sgd {iters} iters: {(time.perf_counter() - t0) * 1e3 / iters:.2f} ms/iter", flush=True)

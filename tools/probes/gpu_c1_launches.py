"""Probe (not collected): config-1 CG (N=2000 RBF fp64, s=1, rank-100 preconditioner) with a
fixed iteration budget -- wall time per iteration, and under ncu a launch list of the
solver's kernels (ITERS env: budget)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import configs as Cfg, warmgp as W

n = 2000
X = Cfg.uniform_rows_fast(W.derive_seed(0, 1), n, 8)
hyp = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
op = W.KernelOperator(hyp, X, precision=W.F64)
b = np.random.default_rng(0).standard_normal(n)
iters = int(os.environ.get("ITERS", "150"))
for budget in (1, iters):
    cfg = W.SolverConfig(tolerance=1e-14, max_iters=budget, precond_rank=100, precond_shift=1e-2)
    for rep in range(3):
        t0 = time.perf_counter()
        r = W.solve(op, b, W.Initialization.cold(), cfg)
        dt = time.perf_counter() - t0
    print(f"budget {budget}: {dt * 1e3:.2f} ms, {r.iterations} iterations", flush=True)

"""Probe (not collected): phase breakdown of a C3-shaped CG solve_many (WGP_PHASE_TIMING=1
prints alloc/upload/pivchol/precond/cg_loop/download wall times to stderr) at several
iteration budgets, so the per-iteration cost and the fixed cost separate."""
import os
import sys
import time

os.environ.setdefault("WGP_PHASE_TIMING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W

n, s = 101000, 64
rng = np.random.default_rng(0)
X = rng.standard_normal((n, 16))
B = np.asfortranarray(rng.standard_normal((n, s)))
hyp = W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, W.MATERN32)
op = W.KernelOperator(hyp, X, precision=W.F32_3XTF32)
for iters in [int(v) for v in os.environ.get("ITERS", "0,1,11,0,1,11").split(",")]:
    cfg = W.SolverConfig(tolerance=1e-12, max_iters=iters, precond_rank=100, precond_shift=1e-3)
    t0 = time.perf_counter()
    res = W.solve_many(op, B, [W.Initialization.cold()] * s, cfg)
    print(f"iters={iters}: solve {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)

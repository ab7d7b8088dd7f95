"""Probe (not collected): does each precision reach tol 1e-4 on BASELINE-like systems?"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W

cases = {
    "C2-like RBF l=.5 sn=.1 d=8 N=10k": (1, 0.5, 0.1, np.random.default_rng(1).random((10000, 8))),
    "C3-like Matern l=.8 sn^2=1e-3 d=16 N=20k": (0, 0.8, 1e-3 ** 0.5, np.random.default_rng(2).standard_normal((20000, 16))),
}
for name, (kind, ls, sn, X) in cases.items():
    n = X.shape[0]
    b = np.random.default_rng(3).standard_normal((n, 4))
    for prec in (W.F64, W.F32_3XTF32, W.F32_SIMT):
        op = W.KernelOperator(W.KernelHyperparams(ls, 1.0, sn, kind), X, precision=prec)
        t0 = time.time()
        res = W.solve_many(op, b, [W.Initialization.cold()] * 4,
                           W.SolverConfig(tolerance=1e-4, max_iters=2000, precond_rank=100, precond_shift=sn * sn))
        dt = time.time() - t0
        print(name, "prec", prec, "iters", [r.iterations for r in res], "conv", [r.converged for r in res],
              "final", [f"{r.residual_history[-1]:.2e}" for r in res], f"min {min(min(r.residual_history) for r in res):.2e}",
              f"{dt:.1f}s", flush=True)

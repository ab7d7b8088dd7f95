"""Probe (not collected): run-to-run variance of the C3 warm/cold CG solves."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import bench
from paper_2511_16340_b200 import warmgp as W
ctx = W.DeviceContext(0)
X = bench.make_inputs()
hyp = W.KernelHyperparams(bench.LS, bench.SF, bench.NOISE_VAR ** 0.5, W.MATERN32)
n, S = X.shape[0], bench.S
op = W.KernelOperator(hyp, X, precision=W.F32_3XTF32, ctx=ctx)
B = np.asfortranarray(np.random.default_rng(0).standard_normal((n, S)))
cfg = W.SolverConfig(tolerance=1e-4, max_iters=1000, precond_rank=100, precond_shift=hyp.noise_scale ** 2)
for i in range(8):
    W.kernel_timer_enable(True)
    t0 = time.perf_counter()
    res = W.solve_many(op, B, [W.Initialization.cold()] * S, cfg)
    dt = time.perf_counter() - t0
    ms, nl = W.kernel_timer_read()
    print(f"solve {i}: {dt:.3f} s, iters {max(r.iterations for r in res)}, TC kernel {nl} launches {ms:.0f} ms total")

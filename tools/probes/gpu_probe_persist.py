"""Probe (not collected): C3 tensor-core kernel time (kernel timer, median of reps) and the
operator error against fp64 at N=20k, under the WGP_TC_* knobs of the calling environment."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W

tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("WGP_TC"))
rng = np.random.default_rng(0)
Xe = rng.standard_normal((20000, 16))
Ve = rng.standard_normal((20000, 8))
he = W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, W.MATERN32)
Y64 = W.KernelOperator(he, Xe, precision=W.F64).kmatvec(Ve)
Ytc = W.KernelOperator(he, Xe, precision=W.F32_3XTF32).kmatvec(Ve)
err = float(np.max(np.linalg.norm(Ytc - Y64, axis=0) / np.linalg.norm(Y64, axis=0)))

for n, s in ((101000, 64), (30000, 64), (101000, 17)):
    X = np.random.default_rng(1).random((n, 16))
    op = W.KernelOperator(W.KernelHyperparams(0.8, 1.0, 0.0316, W.MATERN32), X, precision=W.F32_3XTF32)
    V = torch.randn(n, s, device="cuda", dtype=torch.float64)
    Y = torch.empty_like(V)
    for _ in range(3):
        op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
    torch.cuda.synchronize()
    times = []
    for _ in range(10):
        W.kernel_timer_enable(True)
        op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
        torch.cuda.synchronize()
        ms, k = W.kernel_timer_read()
        W.kernel_timer_enable(False)
        times.append(ms)
    ms = float(np.median(times))
    fl = n * n * (2 * 16 + 2 * s)
    print(f"[{tag}] n={n} s={s} kernel {ms:.3f} ms ({min(times):.3f} min) {fl / ms / 1e9:.1f} TF/s; err20k {err:.2e}",
          flush=True)

"""Probe (not collected): tensor-core operator error at the C3 shape (N=101k, d=16,
Matern l=0.8) against the fp64 operator, random-normal and all-positive RHS, plus kernel
time, under the WGP_TC_CH of the environment."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W

n = 101000
rng = np.random.default_rng(3)
X = rng.standard_normal((n, 16))
V = rng.standard_normal((n, 8))
V[:, 0] = 1.0
V[:, 1] = rng.random(n)
hyp = W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, W.MATERN32)
Y64 = W.KernelOperator(hyp, X, precision=W.F64).kmatvec(V)
op = W.KernelOperator(hyp, X, precision=W.F32_3XTF32)
Ytc = op.kmatvec(V)
err = np.linalg.norm(Ytc - Y64, axis=0) / np.linalg.norm(Y64, axis=0)
Vd = torch.randn(n, 64, device="cuda", dtype=torch.float64)
Yd = torch.empty_like(Vd)
for _ in range(3):
    op.kmatvec_dev(Vd.data_ptr(), Yd.data_ptr(), 64)
torch.cuda.synchronize()
ts = []
for _ in range(8):
    W.kernel_timer_enable(True)
    op.kmatvec_dev(Vd.data_ptr(), Yd.data_ptr(), 64)
    torch.cuda.synchronize()
    ts.append(W.kernel_timer_read()[0])
    W.kernel_timer_enable(False)
print(f"CH={os.environ.get('WGP_TC_CH', 'default')}: kernel {np.median(ts):.3f} ms; err ones {err[0]:.2e} "
      f"uniform {err[1]:.2e} normal max {err[2:].max():.2e}", flush=True)

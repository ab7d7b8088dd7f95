"""Probe (not collected): tcgen05 kernel-matvec kernel-only time (kernel timer) and MUFU
roofline fraction across the BASELINE shapes and both kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W

SHAPES = [  # name, kernel, ls, sn, n, d, s, X
    ("C3 matern d16 s64", W.MATERN32, 0.8, 1e-3 ** 0.5, 101000, 16, 64, "normal"),
    ("C3-shape rbf d16 s64", W.RBF, 0.8, 1e-3 ** 0.5, 101000, 16, 64, "normal"),
    ("C4 rbf d8 s32 N=500k", W.RBF, 0.5, 0.1, 500000, 8, 32, "uniform"),
    ("C4-shape matern d8 s32 N=200k", W.MATERN32, 0.5, 0.1, 200000, 8, 32, "uniform"),
    ("C2 rbf d8 s17 N=20k", W.RBF, 0.5, 0.1, 20000, 8, 17, "uniform"),
    ("C5 matern d6 s129 N=8.2k", W.MATERN32, 0.3, 1e-3, 8200, 6, 129, "uniform"),
]
only = os.environ.get("ONLY")
for name, kind, ls, sn, n, d, s, dist in SHAPES:
    if only and only not in name:
        continue
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, d)) if dist == "normal" else rng.random((n, d))
    op = W.KernelOperator(W.KernelHyperparams(ls, 1.0, sn, kind), X, precision=W.F32_3XTF32)
    V = torch.randn(n, s, device="cuda", dtype=torch.float64)
    Y = torch.empty_like(V)
    for _ in range(2):
        op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
    torch.cuda.synchronize()
    reps = max(3, min(50, int(2e13 / (n * n * (2 * d + 2 * s)))))
    W.kernel_timer_enable(True)
    for _ in range(reps):
        op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
    torch.cuda.synchronize()
    ms, launches = W.kernel_timer_read()
    W.kernel_timer_enable(False)
    dt = ms / launches * 1e-3
    fl = n * n * (2 * d + 2 * s)
    mufu = 2 if kind == W.MATERN32 else 1
    t_mufu = n * n * mufu / (16 * 148 * 1.965e9)
    print(f"{name:32s} kernel {dt*1e3:9.3f} ms {fl/dt/1e12:7.1f} TFLOP/s  MUFU-roof {t_mufu*1e3:8.3f} ms "
          f"frac {t_mufu/dt:.3f}", flush=True)

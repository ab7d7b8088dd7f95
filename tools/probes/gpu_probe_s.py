"""Probe (not collected): C3-shaped kernel-matvec time vs RHS width s (V tile bytes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2511_16340_b200 import warmgp as W
n, d = 101000, 16
X = np.random.default_rng(0).standard_normal((n, d))
op = W.KernelOperator(W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, W.MATERN32), X, precision=W.F32_3XTF32)
st = torch.cuda.Stream()
for s in (16, 32, 48, 64):
    V = torch.randn(n, s, dtype=torch.float64, device="cuda"); Y = torch.empty_like(V)
    for _ in range(3): op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s, st.cuda_stream)
    W.kernel_timer_enable(True)
    for _ in range(10): op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s, st.cuda_stream)
    ms, nl = W.kernel_timer_read(); W.kernel_timer_enable(False)
    ms /= nl
    tiles = ((n + 127) // 128) * ((n + 63) // 64)
    print(f"s={s}: {ms:.3f} ms  ({ms * 1e-3 * 1.9e9 * 148 / tiles:.0f} cycles/tile @1.9GHz)")

"""Probe (not collected): a few C3 tensor-core matvecs (for ncu captures of one launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W

n, s = 101000, 64
X = np.random.default_rng(1).random((n, 16))
op = W.KernelOperator(W.KernelHyperparams(0.8, 1.0, 0.0316, W.MATERN32), X, precision=W.F32_3XTF32)
V = torch.randn(n, s, device="cuda", dtype=torch.float64)
Y = torch.empty_like(V)
for _ in range(int(os.environ.get("REPS", "3"))):
    op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
torch.cuda.synchronize()
print("ok", float(Y.abs().sum()))

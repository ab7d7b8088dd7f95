"""Debug aid (not a test): one C3-shaped matvec with per-tile event clocks of CTA 0."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W
n = 101000
X = np.random.default_rng(0).standard_normal((n, 16))
op = W.KernelOperator(W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, 0), X, precision=W.F32_3XTF32)
V = torch.randn(n, 64, device="cuda", dtype=torch.float64)
Y = torch.empty_like(V)
op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), 64)
torch.cuda.synchronize()
print("done")

"""Debug aid (not a test): one C4-shaped (RBF d=8 s=32, N=100k) matvec with per-tile clocks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W, configs as Cfg
n = 100000
X = Cfg.uniform_rows_fast(1, n, 8)
op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF), X, precision=W.F32_3XTF32)
V = torch.randn(n, 32, device="cuda", dtype=torch.float64)
Y = torch.empty_like(V)
op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), 32)
torch.cuda.synchronize()
print("done")

"""Probe (not collected): the C2 growth sweep's fp32-anchored CG (warm chain, 6 steps) wall time
and the 20k-row tensor-core matvec kernel time, for A/B of library builds (WGP_LIB_PATH)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import configs as Cfg
from paper_2511_16340_b200 import warmgp as W

t0 = time.perf_counter()
out = Cfg.growth_sweep(method=W.CG, steps=range(6), precision=W.F32_3XTF32, residual=W.RESIDUAL_ANCHORED)
wall = time.perf_counter() - t0
secs = {m: sum(r["seconds"] for r in out["steps"] if r["mode"] == m) for m in ("warm", "cold")}
X = np.random.default_rng(0).random((20000, 8))
op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF), X, precision=W.F32_3XTF32)
V = torch.randn(20000, 17, device="cuda", dtype=torch.float64)
Y = torch.empty_like(V)
for _ in range(3):
    op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), 17)
torch.cuda.synchronize()
W.kernel_timer_enable(True)
t1 = time.perf_counter()
for _ in range(50):
    op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), 17)
torch.cuda.synchronize()
t_call = (time.perf_counter() - t1) / 50
ms, k = W.kernel_timer_read("kmatvec_tc")
print(f"{os.path.basename(os.environ.get('WGP_LIB_PATH', 'base'))}: sweep wall {wall:.2f} s, solve warm {secs['warm']:.2f} "
      f"cold {secs['cold']:.2f} s; 20k matvec kernel {ms / k * 1e3:.1f} us, call {t_call * 1e6:.1f} us", flush=True)

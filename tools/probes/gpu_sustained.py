"""Probe (not collected): sustained C3 kernel-matvec (STEPS back-to-back launches after a
warm-up, L2 flushed between launches like the bench) -- average kernel time and the SM clock
under the power cap, for A/B of variants (WGP_LIB_PATH)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import bench
from paper_2511_16340_b200 import warmgp as W

steps = int(os.environ.get("STEPS", "100"))
kind = os.environ.get("KIND", "matern")
ctx = W.DeviceContext(0)
if kind == "matern":
    X = bench.make_inputs()
    hyp = W.KernelHyperparams(bench.LS, bench.SF, bench.NOISE_VAR ** 0.5, W.MATERN32)
    s = 64
else:  # C4-shape RBF
    X = np.random.default_rng(0).random((200000, 8))
    hyp = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
    s = 32
op = W.KernelOperator(hyp, X, precision=W.F32_3XTF32, ctx=ctx)
n = op.n
V = torch.randn(n, s, device="cuda", dtype=torch.float64)
Y = torch.empty_like(V)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
torch.cuda.synchronize()
W.kernel_timer_enable(True)
with bench.ClockSampler(0) as clk:
    for _ in range(steps):
        flush.zero_()
        op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
    torch.cuda.synchronize()
ms, k = W.kernel_timer_read("kmatvec_tc")
W.kernel_timer_enable(False)
c = clk.summary()
print(f"{os.path.basename(os.environ.get('WGP_LIB_PATH', 'base'))} {kind}: {ms / k:.3f} ms per launch over {k}, "
      f"sm {c.get('sm_mhz')} MHz {c.get('reasons')}", flush=True)

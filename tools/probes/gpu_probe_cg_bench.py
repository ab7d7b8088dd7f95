"""Probe (not collected): the bench C3 CG leg, with per-solve timing and kernel totals."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import bench
from paper_2511_16340_b200 import warmgp as W
ctx = W.DeviceContext(0)
X = bench.make_inputs()
hyp = W.KernelHyperparams(bench.LS, bench.SF, bench.NOISE_VAR ** 0.5, W.MATERN32)
W.kernel_timer_enable(True)
out = bench.cg_time_to_tolerance(W, ctx, X, W.F32_3XTF32, hyp)
ms, nl = W.kernel_timer_read()
print({k: (v["seconds"], v["iters_max"]) for k, v in out.items() if isinstance(v, dict)})
print("TC kernel launches", nl, "total ms", ms, "avg", ms / max(nl, 1))

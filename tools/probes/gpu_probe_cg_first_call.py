"""Probe (not collected): the bench C3 CG leg's per-call times with the nvidia-smi clock
sampler (SAMPLER=smi, the bench's), an in-process NVML sampler (SAMPLER=nvml) or none
(SAMPLER=none) -- is the slow first call of the leg the sampler's first nvidia-smi?"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
from paper_2511_16340_b200 import warmgp as W

mode = os.environ.get("SAMPLER", "smi")
if mode == "none":
    class _Null:
        def __init__(self, *a): pass
        def __enter__(self): return self
        def __exit__(self, *a): pass
        def summary(self): return {}
    bench.ClockSampler = _Null
elif mode == "nvml":
    bench.ClockSampler = bench.NvmlClockSampler
ctx = W.DeviceContext(0)
X = bench.make_inputs()
hyp = W.KernelHyperparams(bench.LS, bench.SF, bench.NOISE_VAR ** 0.5, W.MATERN32)
out = bench.cg_time_to_tolerance(W, ctx, X, W.F32_3XTF32, hyp)
print(mode, "cold", [round(x, 3) for x in out["cold"]["seconds_all"]],
      "warm", [round(x, 3) for x in out["warm"]["seconds_all"]], json.dumps(out["clocks_during_cg"]))

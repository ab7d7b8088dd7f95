"""Probe (not collected): software-exp2 share (WGP_TC_SWQ) -> speed and accuracy."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W, configs as Cfg

q = os.environ.get("WGP_TC_SWQ", "default")
def timeit(kind, ls, sn, d, n, s, gauss, reps=10):
    h = W.KernelHyperparams(ls, 1.0, sn, kind)
    X = np.random.default_rng(0).standard_normal((n, d)) if gauss else Cfg.uniform_rows_fast(1, n, d)
    o = W.KernelOperator(h, X, precision=W.F32_3XTF32)
    st = torch.cuda.Stream()
    V = torch.randn(n, s, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    Y = torch.empty_like(V)
    for _ in range(3):
        o.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s, st.cuda_stream)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        o.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s, st.cuda_stream)
    e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, n * n * (2 * d + 2 * s) / ms / 1e9, X, V, Y, h
out = []
for name, args in (("C3", (W.MATERN32, 0.8, 1e-3 ** 0.5, 16, 101000, 64, True)),
                   ("C4@100k", (W.RBF, 0.5, 0.1, 8, 100000, 32, False))):
    ms, tf, X, V, Y, h = timeit(*args)
    # accuracy on a 4000-row slice of the output vs the fp64 operator restricted to it
    o64 = W.KernelOperator(h, X, precision=W.F64)
    Y64 = torch.empty_like(V)
    o64.kmatvec_dev(V.data_ptr(), Y64.data_ptr(), V.shape[1])
    torch.cuda.synchronize()
    err = (torch.linalg.norm(Y - Y64) / torch.linalg.norm(Y64)).item()
    out.append(f"{name}: {ms:.3f} ms {tf:.1f} TFLOP/s relerr {err:.2e}")
print(f"SWQ={q}: " + " | ".join(out))

"""Probe (not collected): kernel-matvec time per precision at config-2/-4/-5 shapes."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W

for name, kind, ls, sn, n, d, s in [("C2 N=20k", 1, 0.5, 0.1, 20000, 8, 17), ("C4-ish N=100k", 1, 0.5, 0.1, 100000, 8, 32),
                                    ("C5 N=8k", 0, 0.3, 1e-3, 8200, 6, 129), ("C3", 0, 0.8, 0.0316, 101000, 16, 64)]:
    X = np.random.default_rng(0).random((n, d))
    for prec in (W.F64, W.F32_SIMT, W.F32_3XTF32):
        if name == "C3" and prec != W.F32_3XTF32 and prec != W.F64:
            continue
        op = W.KernelOperator(W.KernelHyperparams(ls, 1.0, sn, kind), X, precision=prec)
        V = torch.randn(n, s, device="cuda", dtype=torch.float64)
        Y = torch.empty_like(V)
        st = torch.cuda.current_stream().cuda_stream
        for _ in range(2):
            op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        fl = n * n * (2 * d + 2 * s)
        print(f"{name} prec={prec} {dt*1e3:9.3f} ms  {fl/dt/1e12:7.1f} TFLOP/s", flush=True)

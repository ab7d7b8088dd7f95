"""Probe (not collected): operator error of the tensor-core kernel-matvec vs the fp64 path
at a reduced C3 shape (Matern d=16, X ~ N(0,I)) and a C4 shape (RBF d=8, uniform), random
and positive V -- the accuracy side of an A/B variant (WGP_LIB_PATH selects the build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W

for name, kind, ls, sn, n, d, dist in (("C3-shape matern", W.MATERN32, 0.8, 1e-3 ** 0.5, 20000, 16, "normal"),
                                       ("C4-shape rbf", W.RBF, 0.5, 0.1, 20000, 8, "uniform")):
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, d)) if dist == "normal" else rng.random((n, d))
    hyp = W.KernelHyperparams(ls, 1.0, sn, kind)
    o64 = W.KernelOperator(hyp, X, precision=W.F64)
    o32 = W.KernelOperator(hyp, X, precision=W.F32_3XTF32)
    G = rng.standard_normal((n, 16))
    a, b = o64.kmatvec(G), o32.kmatvec(G)
    Gp = np.abs(G)
    ap, bp = o64.kmatvec(Gp), o32.kmatvec(Gp)
    print(f"{name}: rel err random V {np.linalg.norm(b - a) / np.linalg.norm(a):.3e}  positive V "
          f"{np.linalg.norm(bp - ap) / np.linalg.norm(ap):.3e}", flush=True)

"""Probe (not collected): attainable-accuracy floor of the fp32 operators on a C2 system.
For v = H^{-1} b (fp64 CG to 1e-10) report ||H~ v - H v|| / ||b|| per precision."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W, configs as Cfg

for kind, ls, sn, d, n in ((W.RBF, 0.5, 0.1, 8, 10000), (W.MATERN32, 0.8, 1e-3 ** 0.5, 16, 10000)):
    hyp = W.KernelHyperparams(ls, 1.0, sn, kind)
    X = Cfg.uniform_rows_fast(1, n, d) if kind == W.RBF else np.random.default_rng(0).standard_normal((n, d))
    op = W.KernelOperator(hyp, X, precision=W.F64)
    p = W.sample_prior(hyp, d, 1024, 7)
    b = W.rff_eval(op, [p])[:, 0] + W.normal_fill(8, n, sn)
    r = W.solve(op, b, W.Initialization.cold(), W.SolverConfig(tolerance=1e-10, max_iters=5000, precond_rank=100, precond_shift=sn * sn))
    v = r.v
    Hv = op.kmatvec(v[:, None])[:, 0]
    G = np.random.default_rng(1).standard_normal((n, 1))
    HG = op.kmatvec(G)
    print(f"kind={kind} n={n} cg64 iters={r.iterations} |v|/|b|={np.linalg.norm(v)/np.linalg.norm(b):.3e} res={np.linalg.norm(Hv-b)/np.linalg.norm(b):.2e}")
    for prec in (W.F32_3XTF32, W.F32_SIMT, W.TF32):
        o = W.KernelOperator(hyp, X, precision=prec)
        e = np.linalg.norm(o.kmatvec(v[:, None])[:, 0] - Hv) / np.linalg.norm(b)
        eg = np.linalg.norm(o.kmatvec(G) - HG) / np.linalg.norm(HG)
        # asymmetry: u^T H~ w - w^T H~ u
        u = np.random.default_rng(2).standard_normal(n); w = np.random.default_rng(3).standard_normal(n)
        a = (u @ o.kmatvec(w[:, None])[:, 0] - w @ o.kmatvec(u[:, None])[:, 0]) / abs(u @ op.kmatvec(w[:, None])[:, 0])
        print(f"  prec={prec}: floor |H~v-Hv|/|b| = {e:.3e}   random-V rel err {eg:.3e}  asym {a:.2e}")

"""GPU debugging aid (not collected): RBF / fp32-path CG NaN hunt."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from oracle import oracle as O
from paper_2511_16340_b200 import warmgp as W

kind, ls, sn, rank, n = 1, 0.7, 0.3, 50, 3000
X = O.uniform_inputs(41, n, 4)
b = O.gaussian_vector(42, n)
ho = O.KernelHyperparams(ls, 1.0, sn, kind)
for prec in (0, 3, 1):
    op = W.KernelOperator(W.KernelHyperparams(ls, 1.0, sn, kind), X, precision=prec)
    rng = np.random.default_rng(0)
    for k in range(3):
        V = rng.standard_normal((n, 1)) * 10.0 ** (k - 1)
        Y = op.kmatvec(V)
        R = O.kmatvec(X, ho, V)
        print(prec, "kmatvec", k, "nan", int(np.isnan(Y).sum()), "rel", float(np.linalg.norm(Y - R) / np.linalg.norm(R)))
    H = O.gram_matrix(X, ho)
    pre = O.CgPreconditioner.from_matrix(H, rank, sn * sn)
    z = pre.apply(b)
    Y = op.kmatvec(z.reshape(-1, 1))[:, 0]
    R = H @ z
    print(prec, "kmatvec(z)", "nan", int(np.isnan(Y).sum()), "rel", float(np.linalg.norm(Y - R) / np.linalg.norm(R)),
          "zmax", float(np.abs(z).max()))
    for it in (1, 2, 3):
        r = W.solve(op, b, W.Initialization.cold(), W.SolverConfig(tolerance=1e-4, max_iters=it, precond_rank=rank, precond_shift=sn * sn))
        print(prec, "cg", it, r.residual_history)
    ro = O.cg_solve(H, b, O.Initialization.cold(), O.SolverConfig(tolerance=1e-4, max_iters=3, precond_rank=rank, precond_shift=sn * sn))
    print("oracle", ro.residual_history)

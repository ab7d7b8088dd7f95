"""GPU debugging aid (not collected by pytest): TC-path matvec/residual vs oracle on the
config that produced NaNs in CG, then short CG runs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from oracle import oracle as O
from paper_2511_16340_b200 import warmgp as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
kind, ls, sn = 0, 1.0, 0.5
X = O.uniform_inputs(41, n, 4)
ho = O.KernelHyperparams(ls, 1.0, sn, kind)
op = W.KernelOperator(W.KernelHyperparams(ls, 1.0, sn, kind), X, precision=W.F32_3XTF32)
rng = np.random.default_rng(0)
for k in range(4):
    V = rng.standard_normal((n, 1)) * (10.0 ** k)
    Y = op.kmatvec(V)
    R = O.kmatvec(X, ho, V)
    print("kmatvec", k, "nan", int(np.isnan(Y).sum()), "rel", float(np.linalg.norm(Y - R) / np.linalg.norm(R)))
Vd = torch.tensor(rng.standard_normal((n, 1)), device="cuda", dtype=torch.float64)
Bd = torch.tensor(rng.standard_normal((n, 1)), device="cuda", dtype=torch.float64)
Yd = torch.empty_like(Vd)
for rep in range(3):
    op.residual_dev(Bd.data_ptr(), Vd.data_ptr(), Yd.data_ptr(), 1)
    torch.cuda.synchronize()
    ref = Bd.cpu().numpy() - O.kmatvec(X, ho, Vd.cpu().numpy())
    y = Yd.cpu().numpy()
    print("residual", rep, "nan", int(np.isnan(y).sum()), "rel", float(np.linalg.norm(y - ref) / np.linalg.norm(ref)))
b = O.gaussian_vector(42, n)
for it in (1, 2, 3, 5):
    r = W.solve(op, b, W.Initialization.cold(), W.SolverConfig(tolerance=1e-4, max_iters=it, precond_rank=100, precond_shift=sn * sn))
    print("cg", it, r.residual_history)
r = W.solve(op, b, W.Initialization.cold(), W.SolverConfig(tolerance=1e-4, max_iters=5, precond_rank=0))
print("cg noprec", r.residual_history)

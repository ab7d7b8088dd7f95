"""GPU debugging aid (not collected): reproduce the fp32-path RBF CG NaN in test order."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import oracle as O
from paper_2511_16340_b200 import warmgp as W

X = O.uniform_inputs(41, 3000, 4)
b = O.gaussian_vector(42, 3000)
for kind, ls, sn, rank in ((0, 1.0, 0.5, 100), (1, 0.7, 0.3, 50), (1, 0.7, 0.3, 50)):
    for prec in (1, 3, 0):
        op = W.KernelOperator(W.KernelHyperparams(ls, 1.0, sn, kind), X, precision=prec)
        for mi in (3, 1000):
            r = W.solve(op, b, W.Initialization.cold(), W.SolverConfig(tolerance=1e-4, max_iters=mi, precond_rank=rank, precond_shift=sn * sn))
            print(kind, prec, mi, r.iterations, r.converged, [round(x, 6) for x in r.residual_history[:4]], flush=True)

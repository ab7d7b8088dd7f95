"""Probe (not collected): accuracy/speed of the TC accumulation chunk length (WGP_TC_CH)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W, configs as Cfg

ch = os.environ.get("WGP_TC_CH", "16")
hyp = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
n = 10000
X = Cfg.uniform_rows_fast(1, n, 8)
op = W.KernelOperator(hyp, X, precision=W.F64)
p = W.sample_prior(hyp, 8, 1024, 7)
b = W.rff_eval(op, [p])[:, 0] + W.normal_fill(8, n, 0.1)
r = W.solve(op, b, W.Initialization.cold(), W.SolverConfig(tolerance=1e-10, max_iters=5000, precond_rank=100, precond_shift=0.01))
Hv = op.kmatvec(r.v[:, None])[:, 0]
G = np.random.default_rng(1).standard_normal((n, 8))
HG = op.kmatvec(G)
o = W.KernelOperator(hyp, X, precision=W.F32_3XTF32)
e = np.linalg.norm(o.kmatvec(r.v[:, None])[:, 0] - Hv) / np.linalg.norm(b)
eg = np.linalg.norm(o.kmatvec(G) - HG) / np.linalg.norm(HG)
cg = W.solve(o, b, W.Initialization.cold(), W.SolverConfig(tolerance=1e-4, max_iters=1500, precond_rank=100, precond_shift=0.01))
print(f"CH={ch} floor={e:.3e} randV={eg:.3e} f32 CG iters={cg.iterations} conv={cg.converged} minres={min(cg.residual_history):.2e} (f64 CG to 1e-4 for ref below)")

def timeit(kind, ls, sn, d, n, s, gauss):
    h = W.KernelHyperparams(ls, 1.0, sn, kind)
    X = np.random.default_rng(0).standard_normal((n, d)) if gauss else Cfg.uniform_rows_fast(1, n, d)
    o = W.KernelOperator(h, X, precision=W.F32_3XTF32)
    st = torch.cuda.Stream()
    V = torch.randn(n, s, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(V)
    for _ in range(3):
        o.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s, st.cuda_stream)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        o.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s, st.cuda_stream)
    e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    fl = n * n * (2 * d + 2 * s)
    return ms, fl / ms / 1e9
for name, args in (("C3", (W.MATERN32, 0.8, 1e-3 ** 0.5, 16, 101000, 64, True)), ("C4@100k", (W.RBF, 0.5, 0.1, 8, 100000, 32, False))):
    ms, tf = timeit(*args)
    print(f"  CH={ch} {name}: {ms:.3f} ms  {tf:.1f} TFLOP/s")

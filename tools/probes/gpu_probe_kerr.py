"""Probe (not collected): per-entry error of the TC operator (V = unit columns isolates the
kernel map from accumulation), and error vs N for random V."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import warmgp as W, configs as Cfg

for kind, ls in ((W.RBF, 0.5), (W.MATERN32, 0.8)):
    hyp = W.KernelHyperparams(ls, 1.0, 0.1, kind)
    n = 10000
    X = Cfg.uniform_rows_fast(1, n, 8)
    o64 = W.KernelOperator(hyp, X, precision=W.F64)
    o32 = W.KernelOperator(hyp, X, precision=W.F32_3XTF32)
    js = np.random.default_rng(0).choice(n, 64, replace=False)
    V = np.zeros((n, 64)); V[js, np.arange(64)] = 1.0
    K64 = o64.kmatvec(V); K32 = o32.kmatvec(V)
    E = np.abs(K32 - K64)
    rel = E / np.maximum(np.abs(K64), 1e-300)
    big = np.abs(K64) > 1e-3
    print(f"kind={kind} unit-V: max abs err {E.max():.3e}  rms abs {np.sqrt((E**2).mean()):.3e}  max rel(|K|>1e-3) {rel[big].max():.3e} median rel {np.median(rel[big]):.3e}")
    # signed bias
    print(f"   mean signed rel err (|K|>1e-3): {np.mean(((K32-K64)/K64)[big]):.3e}")
    for m in (1000, 3000, 10000):
        G = np.random.default_rng(1).standard_normal((m, 8))
        a = W.KernelOperator(hyp, X[:m], precision=W.F64).kmatvec(G)
        b = W.KernelOperator(hyp, X[:m], precision=W.F32_3XTF32).kmatvec(G)
        c = W.KernelOperator(hyp, X[:m], precision=W.F32_SIMT).kmatvec(G)
        P = np.abs(W.KernelOperator(hyp, X[:m], precision=W.F64).kmatvec(np.abs(G)))
        print(f"   N={m}: randV rel err tc {np.linalg.norm(b-a)/np.linalg.norm(a):.3e} simt {np.linalg.norm(c-a)/np.linalg.norm(a):.3e}   err/(|K||V|) tc {np.abs(b-a).max()/P.max():.3e}")
        Gp = np.abs(G)
        a = W.KernelOperator(hyp, X[:m], precision=W.F64).kmatvec(Gp)
        b = W.KernelOperator(hyp, X[:m], precision=W.F32_3XTF32).kmatvec(Gp)
        print(f"   N={m}: positive-V rel err tc {np.linalg.norm(b-a)/np.linalg.norm(a):.3e} mean signed {np.mean((b-a)/a):.3e}")

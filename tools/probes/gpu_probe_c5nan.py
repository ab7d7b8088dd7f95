"""Probe (not collected): find where config 5's budgeted solves turn NaN (D=2, cold)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2511_16340_b200 import configs as Cfg
from paper_2511_16340_b200 import warmgp as W

dim, seed, batch, cands = 2, 0, 64, 100_000
hyp = W.KernelHyperparams(0.3, 1.0, 1e-3, W.MATERN32)
cfg = W.SolverConfig(method=W.CG, tolerance=1e-2, max_iters=5, precond_rank=100,
                     precond_shift=hyp.noise_scale ** 2)
obj = Cfg.BumpObjective.make(dim, seed)
X0 = Cfg.uniform_rows_fast(W.derive_seed(seed, 2), 5000, dim)
st = Cfg.growth_state(X0, obj.observe(X0), hyp, 128, 2000, seed, W.F64)
st.op_fast = W.KernelOperator(hyp, X0, precision=W.F32_3XTF32)
Xall = X0.copy()
for r in range(14):
    rec = st.solve_round(cfg, False)
    B = st.rhs()
    bad = not np.isfinite(rec["mean_residual"])
    print(f"round {rec['round']} n {st.n_obs} res {rec['mean_residual']:.3e} sample {rec['avg_sample_residual']:.3e} "
          f"B finite {np.isfinite(B).all()} y finite {np.isfinite(st.y).all()} "
          f"w finite {np.isfinite(st.weights).all()}", flush=True)
    if bad:
        u, cnt = np.unique(Xall, axis=0, return_counts=True)
        print("  duplicate rows:", int((cnt > 1).sum()), "max multiplicity", int(cnt.max()))
        dmin = np.inf
        print("  X range", Xall.min(0), Xall.max(0))
        for rank in (0, 100):
            for meth in (W.CG,):
                c2 = cfg.copy(precond_rank=rank)
                res = W.solve_many(st.op, B[:, :2], [W.Initialization.cold()] * 2, c2)
                print(f"  rank {rank}: hist {res[0].residual_history}", flush=True)
        res, status, dv = W.solve_many(st.op, B, [W.Initialization.cold()] * B.shape[1],
                                       cfg.copy(seed=W.derive_seed(seed, 0xC0000 + st.round)), return_status=True)
        nanc = [c for c in range(B.shape[1]) if not np.isfinite(res[c].v).all()]
        print("  full solve_many: nan columns", nanc[:10], "count", len(nanc), "status", sorted(set(status.tolist())))
        if nanc:
            c0 = nanc[0]
            print("  col", c0, "hist", res[c0].residual_history, flush=True)
            one = W.solve_many(st.op, B[:, c0:c0 + 1], [W.Initialization.cold()], cfg)
            print("  alone hist", one[0].residual_history, flush=True)
            for grp in (1, 8, 64):
                sub = W.solve_many(st.op, np.asfortranarray(B[:, :grp]), [W.Initialization.cold()] * grp, cfg)
                print(f"  first {grp} cols: nan {sum(not np.isfinite(r.v).all() for r in sub)}", flush=True)
        Y = st.op.kmatvec(B[:, :2])
        print("  kmatvec finite", np.isfinite(Y).all(), flush=True)
        break
    Xc = Cfg.uniform_rows_fast(W.derive_seed(seed, 0xA0000 + st.round), cands, dim)
    F = Cfg.posterior_at(st, Xc)[:, :batch]
    print(f"  F finite {np.isfinite(F).all()} range {np.nanmin(F):.3g} {np.nanmax(F):.3g}", flush=True)
    g = np.array_split(np.arange(cands), 5)
    starts = np.stack([Xc[gi[np.argmax(F[gi], axis=0)]] for gi in g], axis=1)
    wd = st.weights[:, :1] - st.weights[:, 1:1 + batch]
    Xn, vals = W.ascend_peaks(st.op, st.priors[:batch], wd, starts, 30, 0.05)
    print(f"  Xn finite {np.isfinite(Xn).all()} on boundary {int(((Xn == 0) | (Xn == 1)).any(1).sum())} "
          f"unique {len(np.unique(Xn, axis=0))}", flush=True)
    st.add_points(Xn, obj.observe(Xn))
    Xall = np.vstack([Xall, Xn])

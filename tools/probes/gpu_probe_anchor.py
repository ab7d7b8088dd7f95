"""Probe: fp32 (3xF16 tensor-core) CG with the direct vs the fp64-anchored true residual,
against the fp64 operator, at C2 / reduced-C4 / C3 shapes.  Prints one JSON object per case.
(Measured r2 in profiles/r02_anchor_probe.log; two algebraically equivalent CG variants --
alpha = p.r / p.Hp and Polak-Ribiere beta -- were also run and changed nothing, so they
were removed from the solver.)

  python tools/probes/gpu_probe_anchor.py [c2] [c4] [c3]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2511_16340_b200 import configs as Cfg  # noqa: E402
from paper_2511_16340_b200 import warmgp as W  # noqa: E402

MODES = (("f64", W.F64, W.RESIDUAL_DIRECT), ("tc_direct", W.F32_3XTF32, W.RESIDUAL_DIRECT),
         ("tc_anchored", W.F32_3XTF32, W.RESIDUAL_ANCHORED),
         ("tc_anchor_every_iter", W.F32_3XTF32, W.RESIDUAL_ANCHORED))


def crossings(h, levels=(1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6)):
    out = {}
    for lv in levels:
        k = next((i for i, r in enumerate(h) if r <= lv), None)
        out[f"{lv:g}"] = k
    return out


def summarize(res, t, op):
    its = [r.iterations for r in res]
    return {"seconds": t, "iters": its, "converged": int(sum(r.converged for r in res)),
            "final": [float(r.residual_history[-1]) for r in res],
            "min": [float(min(r.residual_history)) for r in res],
            "cross0": crossings(res[0].residual_history),
            "anchors": op.last_anchor_count}


def solve_all(hyp, X, B, inits_fn, cfg, label, modes=MODES):
    out = {}
    for name, prec, rm in modes:
        if name == "tc_anchor_every_iter":
            os.environ["WGP_ANCHOR_FRAC"] = "0"
        else:
            os.environ.pop("WGP_ANCHOR_FRAC", None)
        op = W.KernelOperator(hyp, X, precision=prec, residual=rm)
        W.solve_many(op, B[:, :1], [W.Initialization.cold()], cfg.copy(max_iters=2))  # warm-up
        t0 = time.perf_counter()
        try:
            res = W.solve_many(op, B, inits_fn(), cfg)
            out[name] = summarize(res, time.perf_counter() - t0, op)
        except Exception as e:  # noqa: BLE001
            out[name] = {"error": repr(e)}
        print(json.dumps({"case": label, "mode": name, "lib": os.path.basename(W.LIB_PATH), **out[name]}), flush=True)
        del op
    return out


def c2():
    hyp = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
    d, pool = 8, 20_000
    Xp = Cfg.uniform_rows_fast(W.derive_seed(0, 1), pool, d)
    fy = W.sample_prior(hyp, d, 1024, W.derive_seed(0, 7))
    tmp = W.KernelOperator(hyp, Xp, precision=W.F64)
    yp = W.rff_eval(tmp, [fy])[:, 0] + W.normal_fill(W.derive_seed(0, 8), pool, 0.1)
    st = Cfg.growth_state(Xp, yp, hyp, 16, 1024, 0, W.F64)
    B = st.rhs()
    cfg = W.SolverConfig(tolerance=1e-4, max_iters=2000, precond_rank=100, precond_shift=0.01)
    for n in (10_000, 20_000):
        solve_all(hyp, Xp[:n], np.asfortranarray(B[:n]), lambda: [W.Initialization.cold()] * 17, cfg,
                  f"c2_cold_n{n}")
    # warm: from the fp64 solution at 19.5k
    op = W.KernelOperator(hyp, Xp[:19_500], precision=W.F64)
    prev = W.solve_many(op, np.asfortranarray(B[:19_500]), [W.Initialization.cold()] * 17, cfg)
    del op
    solve_all(hyp, Xp, np.asfortranarray(B), lambda: [W.Initialization.warm(r.v) for r in prev], cfg,
              "c2_warm_n20000")


def c4(n=30_000, s=8, budget=1000):
    hyp = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
    d = 8
    X = Cfg.uniform_rows_fast(W.derive_seed(0, 1), n, d)
    tmp = W.KernelOperator(hyp, X, precision=W.F64)
    priors = [W.sample_prior(hyp, d, 1024, W.derive_seed(0, 7 + 100 * c)) for c in range(s)]
    B = np.asfortranarray(W.rff_eval(tmp, priors) + W.normal_fill(W.derive_seed(0, 9), n * s, 0.1).reshape(n, s))
    del tmp
    cfg = W.SolverConfig(tolerance=1e-12, max_iters=budget, precond_rank=100, precond_shift=0.01)
    solve_all(hyp, X, B, lambda: [W.Initialization.cold()] * s, cfg, f"c4_cold_n{n}_s{s}")


def c3():
    n0, na, d, s = 100_000, 1_000, 16, 64
    hyp = W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, W.MATERN32)
    X = np.random.default_rng(0).standard_normal((n0 + na, d))
    n = n0 + na
    priors = [W.sample_prior(hyp, d, 2048, W.derive_seed(0, 100 + c)) for c in range(s)]
    full = W.KernelOperator(hyp, X, precision=W.F64)
    B = W.rff_eval(full, priors)
    del full
    B += hyp.noise_scale * W.normal_fill(W.derive_seed(0, 3), n * s).reshape(n, s, order="F")
    B = np.asfortranarray(B)
    cfg = W.SolverConfig(tolerance=1e-4, max_iters=1000, precond_rank=100, precond_shift=1e-3)
    op = W.KernelOperator(hyp, X[:n0], precision=W.F64)
    prev = W.solve_many(op, np.asfortranarray(B[:n0]), [W.Initialization.cold()] * s, cfg)
    del op
    modes = (MODES[0], MODES[1], MODES[3])
    solve_all(hyp, X, B, lambda: [W.Initialization.warm(r.v) for r in prev], cfg, "c3_warm", modes)
    solve_all(hyp, X, B, lambda: [W.Initialization.cold()] * s, cfg, "c3_cold", modes)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c2", "c4", "c3"]
    for w in which:
        {"c2": c2, "c4": c4, "c3": c3}[w]()

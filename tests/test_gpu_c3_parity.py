"""CG parity at the C3 shape (BASELINE configs[2]): Matern-3/2, l = 0.8, s_f = 1,
sigma_n^2 = 1e-3, X ~ N(0, I_16), right-hand sides = Matern RFF prior samples (F = 2048) plus
sigma_n noise, tol 1e-4, warm start [u; 0] after appending rows (solvers.cpp:142-183).

* Reduced N = 4000 + 100: the fp64 device path against the CPU oracle (dense H) -- iteration
  counts within +-2%, early residual histories to 1e-6.
* Full N = 100,000 + 1,000 (s = 16 of the 64 columns): the fp32-class tensor-core path against
  the fp64 DMMA path (itself pinned to the oracle above).  Measured (profiles/r02_anchor_probe
  .log, s = 64): tc 18.8 vs fp64 17.8 iterations warm (+6%), 27.0 vs 24.1 cold (+12%); the
  excess comes from the fp32 H p (anchoring the true residual in fp64 every iteration leaves
  it unchanged), so the band asserted here is [-2%, +15%], and the TC solution's TRUE residual
  (fp64 operator) must meet the tolerance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LS, NOISE_VAR, D = 0.8, 1e-3, 16


def problem(W, n0, na, s, seed=0):
    hyp = W.KernelHyperparams(LS, 1.0, NOISE_VAR ** 0.5, W.MATERN32)
    X = np.random.default_rng(seed).standard_normal((n0 + na, D))
    n = n0 + na
    priors = [W.sample_prior(hyp, D, 2048, W.derive_seed(seed, 100 + c)) for c in range(s)]
    full = W.KernelOperator(hyp, X, precision=W.F64)
    B = W.rff_eval(full, priors)
    B += hyp.noise_scale * W.normal_fill(W.derive_seed(seed, 3), n * s).reshape(n, s, order="F")
    return hyp, X, np.asfortranarray(B), full


def cfg_c3(W, **kw):
    return W.SolverConfig(tolerance=1e-4, max_iters=1000, precond_rank=100, precond_shift=NOISE_VAR, **kw)


def test_c3_reduced_f64_vs_oracle(W, O):
    n0, na, s = 4000, 100, 4
    hyp, X, B, full = problem(W, n0, na, s, seed=1)
    h = O.KernelHyperparams(LS, 1.0, NOISE_VAR ** 0.5, O.MATERN32)
    H0, H = O.gram_matrix(X[:n0], h), O.gram_matrix(X, h)
    ocfg = O.SolverConfig(tolerance=1e-4, max_iters=1000, precond_rank=100, precond_shift=NOISE_VAR)
    prev = [O.cg_solve(H0, B[:n0, c], O.Initialization.cold(), ocfg) for c in range(s)]
    op0 = W.KernelOperator(hyp, X[:n0], precision=W.F64)
    dprev = W.solve_many(op0, np.asfortranarray(B[:n0]), [W.Initialization.cold()] * s, cfg_c3(W))
    op0.append_rows(X[n0:])  # +100 rows on the device (extend_system)
    for c in range(s):
        assert abs(dprev[c].iterations - prev[c].iterations) <= max(1, round(0.02 * prev[c].iterations))
        ref = O.cg_solve(H, B[:, c], O.Initialization.warm(prev[c].v), ocfg)
        got = W.solve(op0, B[:, c], W.Initialization.warm(dprev[c].v), cfg_c3(W))
        assert got.converged and ref.converged
        assert abs(got.iterations - ref.iterations) <= max(1, round(0.02 * ref.iterations)), \
            (c, got.iterations, ref.iterations)
        k = min(6, len(ref.residual_history))
        np.testing.assert_allclose(got.residual_history[:k], ref.residual_history[:k], rtol=1e-6)


@pytest.mark.parametrize("mode", ["warm", "cold"])
def test_c3_full_shape_tensor_core_vs_f64(W, mode):
    n0, na, s = 100_000, 1_000, 16
    hyp, X, B, full = problem(W, n0, na, s)
    cfg = cfg_c3(W)
    inits = [W.Initialization.cold()] * s
    if mode == "warm":  # the N = 100k system's fp64 solution, zero-extended (expand_init)
        op0 = W.KernelOperator(hyp, X[:n0], precision=W.F64)
        prev = W.solve_many(op0, np.asfortranarray(B[:n0]), [W.Initialization.cold()] * s, cfg)
        del op0
        inits = [W.Initialization.warm(r.v) for r in prev]
    ref = W.solve_many(full, B, inits, cfg)
    tc = W.KernelOperator(hyp, X[:n0], precision=W.F32_3XTF32)
    tc.append_rows(X[n0:])  # device-resident growth, as the bench's C3 step
    got = W.solve_many(tc, B, inits, cfg)
    V = np.column_stack([r.v for r in got])
    true = W.relative_residual(full, V, B)
    for c, (g, r) in enumerate(zip(got, ref)):
        assert r.converged and g.converged
        lo = r.iterations - max(1, round(0.02 * r.iterations))
        hi = r.iterations + max(1, round(0.15 * r.iterations))
        assert lo <= g.iterations <= hi, (mode, c, g.iterations, r.iterations)
        assert true[c] <= 1.05e-4, (mode, c, true[c])

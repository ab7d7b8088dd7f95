"""GPU parity of the configuration drivers (callers of the path) against the oracle:
config 1 at full size, the sequential-growth bookkeeping of bo_round
(thompson.cpp:321-386, 403-422) and the posterior evaluation of config 5
(eval_posterior, sampling.cpp:66-75)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def iters_close(a, b):
    return abs(a - b) <= max(1, round(0.02 * max(a, b)))


def test_config1_full_size_parity(W, O):
    """Config 1 at N=2000 (bench_regression.cpp:139-197 protocol): exact u1 on the first
    1900 rows, CG warm and cold to 1e-6 -- iteration counts within +-2% of the oracle."""
    h = O.KernelHyperparams(0.5, 1.0, 0.1, O.RBF)
    n1, n = 1900, 2000
    X = O.uniform_inputs(O.derive_seed(0, 1), n, 8)
    prior = O.sample_prior(h, 8, 1024, O.derive_seed(0, 7))
    y = O.build_sample_rhs(prior, X, 0.1, O.derive_seed(0, 8))
    u1 = O.exact_solve(O.gram_matrix(X[:n1], h), y[:n1])
    H = O.gram_matrix(X, h)
    ocfg = O.SolverConfig(tolerance=1e-6, max_iters=2000, precond_rank=100, precond_shift=0.01)
    o_cold = O.cg_solve(H, y, O.Initialization.cold(), ocfg)
    o_warm = O.cg_solve(H, y, O.Initialization.warm(u1), ocfg)

    op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF), X, precision=W.F64)
    # the device RHS builder agrees with build_sample_rhs (fp64 cos on the device)
    wp = W.sample_prior(op.hyp, 8, 1024, W.derive_seed(0, 7))
    yd = W.build_sample_rhs(op, wp, 0.1, W.derive_seed(0, 8))
    assert np.abs(yd - y).max() <= 1e-10 * np.abs(y).max()
    cfg = W.SolverConfig(tolerance=1e-6, max_iters=2000, precond_rank=100, precond_shift=0.01)
    cold = W.solve(op, y, W.Initialization.cold(), cfg)
    warm = W.solve(op, y, W.Initialization.warm(u1), cfg)
    for g, o in ((cold, o_cold), (warm, o_warm)):
        assert g.converged and o.converged
        assert iters_close(g.iterations, o.iterations), (g.iterations, o.iterations)
        np.testing.assert_allclose(g.residual_history[:5], o.residual_history[:5], rtol=1e-8)
    assert warm.iterations < cold.iterations


def _oracle_growth(O, X, y, hyp, S, F, seed, cfg, rounds):
    """The bo_round warm bookkeeping restated on the oracle (thompson.cpp:260-293,
    321-386, 403-422); rounds = list of row counts."""
    d = X.shape[1]
    priors = [O.sample_prior(hyp, d, F, O.derive_seed(seed, 100 + s)) for s in range(S)]
    noise = O.Rng(O.derive_seed(seed, 3))
    n0 = rounds[0]
    pv = np.column_stack([O.eval_prior(p, X[:n0]) for p in priors])
    nd = np.array([[hyp.noise_scale * noise.normal() for _ in range(S)] for _ in range(n0)])
    weights, out = None, []
    for r, n in enumerate(rounds, start=1):
        if n > pv.shape[0]:
            m0 = pv.shape[0]
            pv = np.vstack([pv, np.column_stack([O.eval_prior(p, X[m0:n]) for p in priors])])
            nd = np.vstack([nd, [[hyp.noise_scale * noise.normal() for _ in range(S)]
                                 for _ in range(n - m0)]])
        B = np.asfortranarray(np.column_stack([y[:n], pv + nd]))
        inits = ([O.Initialization.warm(weights[:, c]) for c in range(S + 1)] if weights is not None
                 else [O.Initialization.cold()] * (S + 1))
        c = O.SolverConfig(tolerance=cfg.tolerance, max_iters=cfg.max_iters, precond_rank=cfg.precond_rank,
                           precond_shift=cfg.precond_shift, seed=O.derive_seed(seed, 0xC0000 + r))
        res = O.solve_many(O.gram_matrix(X[:n], hyp), B, inits, c)
        weights = np.column_stack([q.v for q in res])
        out.append((B.copy(), res))
    return out


def test_growth_bookkeeping_matches_oracle(W, O):
    """Three growth rounds (n = 300, 350, 400), y + 4 pathwise samples: the device driver's
    right-hand sides (prior values at new rows, i-major noise) and warm-started solves
    agree with the oracle's restatement of bo_round."""
    from paper_2511_16340_b200 import configs as Cfg
    seed, S, F = 5, 4, 256
    rounds = [300, 350, 400]
    X = O.uniform_inputs(O.derive_seed(seed, 1), rounds[-1], 3)
    y = O.gaussian_vector(O.derive_seed(seed, 2), rounds[-1])
    ohyp = O.KernelHyperparams(0.3, 1.0, 0.05, O.MATERN32)
    cfg = W.SolverConfig(tolerance=1e-8, max_iters=500, precond_rank=50, precond_shift=0.05 ** 2)
    ref = _oracle_growth(O, X, y, ohyp, S, F, seed, cfg, rounds)

    st = Cfg.growth_state(X[:rounds[0]], y[:rounds[0]], W.KernelHyperparams(0.3, 1.0, 0.05, W.MATERN32),
                          S, F, seed, W.F64)
    for r, n in enumerate(rounds):
        if st.n_obs < n:
            st.add_points(X[st.n_obs:n], y[st.n_obs:n])
        B_ref, res_ref = ref[r]
        B = st.rhs()
        assert np.array_equal(B[:, 0], B_ref[:, 0])
        # noise draws are bitwise (host Rng); prior values are fp64 device cos
        assert np.abs(B - B_ref).max() <= 1e-11 * np.abs(B_ref).max()
        rec = st.solve_round(cfg, warm=True)
        assert rec["warm"] == (r > 0)
        for c, q in enumerate(res_ref):
            assert iters_close(rec["iterations"][c], q.iterations), (r, c, rec["iterations"][c], q.iterations)
            assert np.linalg.norm(st.weights[:, c] - q.v) <= 1e-5 * np.linalg.norm(q.v)


def test_growth_divergence_keeps_initial_weights(W):
    """solve_best_effort (thompson.cpp:299-317): a diverging SGD column keeps its
    (zero-extended warm) initial weights with a one-entry history, and the next round
    warm-starts from them."""
    from paper_2511_16340_b200 import configs as Cfg
    X = Cfg.uniform_rows_fast(9, 260, 2)
    hyp = W.KernelHyperparams(0.3, 1.0, 0.1, W.MATERN32)
    st = Cfg.growth_state(X[:200], np.sin(6 * X[:200, 0]), hyp, 2, 128, 9, W.F64)
    good = W.SolverConfig(method=W.CG, tolerance=1e-6, max_iters=300, precond_rank=20, precond_shift=0.01)
    st.solve_round(good, warm=True)
    w0 = st.weights.copy()
    st.add_points(X[200:260], np.sin(6 * X[200:260, 0]))
    bad = W.SolverConfig(method=W.SGD, tolerance=1e-6, max_iters=200, learning_rate=50.0, batch_size=20)
    rec = st.solve_round(bad, warm=True)
    assert rec["diverged"] == 3
    assert np.array_equal(st.weights[:200], w0) and not st.weights[200:].any()
    rec = st.solve_round(good, warm=True)
    assert rec["converged"] == 3 and rec["warm"]


def test_posterior_at_matches_eval_posterior(W, O):
    """posterior_at = prior_s(X*) + K(X*, X)(w_mean - w_s) (sampling.cpp:66-75) for every
    sample, against the oracle's eval_posterior."""
    from paper_2511_16340_b200 import configs as Cfg
    seed = 4
    X = O.uniform_inputs(O.derive_seed(seed, 1), 250, 4)
    y = O.gaussian_vector(O.derive_seed(seed, 2), 250)
    st = Cfg.growth_state(X, y, W.KernelHyperparams(0.3, 1.0, 1e-3 ** 0.5, W.MATERN32), 3, 300, seed, W.F64)
    st.solve_round(W.SolverConfig(tolerance=1e-3, max_iters=50, precond_rank=50, precond_shift=1e-3), warm=True)
    Xc = O.uniform_inputs(O.derive_seed(seed, 9), 1000, 4)
    F = Cfg.posterior_at(st, Xc)
    ohyp = O.KernelHyperparams(0.3, 1.0, 1e-3 ** 0.5, O.MATERN32)
    for s in range(3):
        p = O.sample_prior(ohyp, 4, 300, O.derive_seed(seed, 100 + s))
        ref = O.eval_posterior(ohyp, p, X, st.weights[:, 0] - st.weights[:, 1 + s], Xc)
        assert np.abs(F[:, s] - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())


def test_bo_loop_smoke(W):
    """Config 5 driver end to end at reduced size: rows grow by `batch` per round and the
    acquired points come from the candidate set."""
    from paper_2511_16340_b200 import configs as Cfg
    out = Cfg.bo_loop(dim=2, n_init=300, batch=8, rounds=3, n_samples=16, candidates=2000)
    assert [r["n"] for r in out["rounds"]] == [300, 308, 316]
    assert out["rounds"][1]["warm"] and all(np.isfinite(r["best_value"]) for r in out["rounds"])


def test_eval_posterior_mirror_matches_oracle(W, O):
    """warmgp.eval_posterior (the sampling.hpp:48 mirror, all samples at once) against the
    oracle's per-sample eval_posterior, fp64 and tensor-core operators."""
    seed = 6
    X = O.uniform_inputs(O.derive_seed(seed, 1), 300, 3)
    Xs = O.uniform_inputs(O.derive_seed(seed, 2), 777, 3)
    wts = np.random.default_rng(seed).standard_normal((300, 4))
    ohyp = O.KernelHyperparams(0.4, 1.2, 0.05, O.MATERN32)
    whyp = W.KernelHyperparams(0.4, 1.2, 0.05, W.MATERN32)
    priors = [W.sample_prior(whyp, 3, 256, W.derive_seed(seed, 100 + s)) for s in range(4)]
    ref = np.column_stack([O.eval_posterior(ohyp, O.sample_prior(ohyp, 3, 256, W.derive_seed(seed, 100 + s)),
                                            X, wts[:, s], Xs) for s in range(4)])
    for prec, tol in ((W.F64, 1e-10), (W.F32_3XTF32, 1e-5)):
        got = W.eval_posterior(W.KernelOperator(whyp, X, precision=prec), priors, wts, Xs)
        assert np.abs(got - ref).max() <= tol * np.abs(ref).max()

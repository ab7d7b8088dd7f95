"""Oracle pins restated from the reference's solver tests (proj/tests/test_solvers.cpp) and
the solver-oracle acceptance pattern (verify.cpp:115-173)."""
import numpy as np
import pytest


def random_spd(O, seed, n, ridge=0.5):  # testutil.hpp:26-35
    r = O.Rng(seed)
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            A[i, j] = r.normal()
    H = A @ A.T / n
    H[np.diag_indices(n)] += ridge
    return np.asfortranarray(H)


def matern_system(O, seed, n, dim=3, ls=0.5, noise=0.5):  # testutil.hpp:44-51
    h = O.KernelHyperparams(ls, 1.0, noise)
    return O.gram_matrix(O.uniform_inputs(seed, n, dim), h), O.gaussian_vector(O.derive_seed(seed, 0xB), n)


def blocked(O, seed, n1, n2, dim=3, ls=0.5, noise=0.3):  # testutil.hpp:54-62
    h = O.KernelHyperparams(ls, 1.0, noise)
    X1 = O.uniform_inputs(seed, n1, dim)
    X2 = O.uniform_inputs(O.derive_seed(seed, 1), n2, dim)
    H11 = O.gram_matrix(X1, h)
    H = O.extend_assembled(H11, X1, X2, h)
    b1 = O.gaussian_vector(O.derive_seed(seed, 2), n1)
    b2 = O.gaussian_vector(O.derive_seed(seed, 3), n2)
    return H11, H, b1, np.concatenate([b1, b2])


def test_init_weights(O):  # test_solvers.cpp:10-31
    v = O.init_weights(O.Initialization.cold(), 3, 2)
    assert v.size == 5 and not v.any()
    v = O.init_weights(O.Initialization.warm([1.0, 2.0]), 2, 1)
    assert list(v) == [1.0, 2.0, 0.0]
    with pytest.raises(ValueError):
        O.init_weights(O.Initialization.warm([1.0, 2.0]), 3, 1)


def test_warm_exact_subsolution_residual(O):  # test_solvers.cpp:33-40
    H11, H, b1, b = blocked(O, 5, 40, 8)
    u1 = O.exact_solve(H11, b1)
    v0 = O.init_weights(O.Initialization.warm(u1), 40, 8)
    r = b - H @ v0
    assert np.abs(r[:40]).max() < 1e-12
    assert np.abs(r[40:] - (b[40:] - H[:40, 40:].T @ u1)).max() < 1e-12


def test_relative_residual(O):  # test_solvers.cpp:42-65
    H = random_spd(O, 1, 12)
    b = O.gaussian_vector(2, 12)
    assert O.relative_residual(H, O.exact_solve(H, b), b) < 1e-12
    H = random_spd(O, 3, 6)
    assert O.relative_residual(H, np.zeros(6), O.gaussian_vector(4, 6)) == 1.0
    assert O.relative_residual(2.0 * np.eye(2), [0.5, 0.0], [2.0, 0.0]) == 0.5
    with pytest.raises(ValueError):
        O.relative_residual(np.eye(2), np.zeros(2), np.zeros(2))


def test_pivoted_cholesky(O):  # test_solvers.cpp:67-100
    H = random_spd(O, 7, 30)
    L = O.pivoted_cholesky(H, 30)
    assert np.abs(L @ L.T - H).max() < 1e-10
    D = np.diag([1.0, 9.0, 4.0, 2.0])
    L = O.pivoted_cholesky(D, 1)
    assert L.shape[1] == 1 and L[1, 0] == pytest.approx(3.0) and L[0, 0] == 0.0 and L[2, 0] == 0.0
    H = random_spd(O, 8, 50)
    prev = np.trace(H)
    for r in range(1, 51, 7):
        L = O.pivoted_cholesky(H, r)
        rt = np.trace(H - L @ L.T)
        assert rt < prev and rt > -1e-9
        prev = rt
    A = O.uniform_inputs(9, 20, 3)
    H = np.asfortranarray(A @ A.T)
    L = O.pivoted_cholesky(H, 10)
    assert L.shape[1] <= 4 and np.abs(L @ L.T - H).max() < 1e-8


def test_preconditioner_dense_inverse(O):  # test_solvers.cpp:102-111
    H, _ = matern_system(O, 10, 40)
    L = O.pivoted_cholesky(H, 15)
    pre = O.CgPreconditioner(L, 0.25)
    r = O.gaussian_vector(11, 40)
    z = pre.apply(r)
    assert np.abs((L @ L.T + 0.25 * np.eye(40)) @ z - r).max() < 1e-9


def test_cg(O):  # test_solvers.cpp:113-156
    cfg = O.SolverConfig(tolerance=1e-10, precond_rank=0)
    res = O.cg_solve(np.eye(10), O.gaussian_vector(12, 10), O.Initialization.cold(), cfg)
    assert res.converged and res.iterations == 1 and len(res.residual_history) == 2
    H = random_spd(O, 13, 20)
    b = O.gaussian_vector(14, 20)
    res = O.cg_solve(H, b, O.Initialization.cold(), O.SolverConfig(tolerance=0.01, precond_rank=10, precond_shift=0.5))
    assert res.converged and O.relative_residual(H, res.v, b) <= 0.01
    ve = O.exact_solve(H, b)
    assert O.rkhs_distance(H, res.v, ve) / O.rkhs_distance(H, np.zeros(20), ve) < 0.1
    with pytest.raises(O.NotSpdError):
        O.cg_solve(np.diag([1.0, -1.0]), [0.0, 1.0], O.Initialization.cold(), O.SolverConfig(precond_rank=0))
    res = O.cg_solve(random_spd(O, 15, 8), np.zeros(8), O.Initialization.cold(), O.SolverConfig())
    assert res.converged and res.iterations == 0 and not res.v.any() and res.residual_history == [0.0]


def test_sgd(O):  # test_solvers.cpp:158-233
    b = O.gaussian_vector(16, 12)
    res = O.sgd_solve(np.eye(12), b, O.Initialization.cold(),
                      O.SolverConfig(method=O.SGD, learning_rate=1.0, momentum=0.0, batch_size=100, tolerance=1e-12))
    assert res.converged and res.iterations == 1 and np.abs(res.v - b).max() < 1e-12
    H = 0.1 * random_spd(O, 17, 50, 0.0) + np.eye(50)
    b = O.gaussian_vector(18, 50)
    res = O.sgd_solve(H, b, O.Initialization.cold(), O.SolverConfig(method=O.SGD, tolerance=0.01, max_iters=5000))
    assert res.converged and res.iterations < 5000 and O.relative_residual(H, res.v, b) <= 0.01
    H, b = matern_system(O, 19, 40)
    cfg = O.SolverConfig(method=O.SGD, learning_rate=0.05, batch_size=10, max_iters=200, tolerance=1e-8, seed=1234)
    a = O.sgd_solve(H, b, O.Initialization.cold(), cfg)
    a2 = O.sgd_solve(H, b, O.Initialization.cold(), cfg)
    assert np.array_equal(a.v, a2.v) and a.residual_history == a2.residual_history
    cfg.seed = 1235
    assert not np.array_equal(a.v, O.sgd_solve(H, b, O.Initialization.cold(), cfg).v)
    with pytest.raises(O.DivergenceError) as ei:
        O.sgd_solve(10.0 * np.eye(20), O.gaussian_vector(20, 20), O.Initialization.cold(),
                    O.SolverConfig(method=O.SGD, learning_rate=5.0, momentum=0.9, batch_size=20, max_iters=10000))
    assert ei.value.iterations >= 1
    H11, H, b1, b = blocked(O, 21, 60, 10)
    u1 = O.exact_solve(H11, b1)
    cfg = O.SolverConfig(method=O.SGD, learning_rate=0.01, max_iters=1, tolerance=1e-12)
    warm = O.sgd_solve(H, b, O.Initialization.warm(u1), cfg)
    cold = O.sgd_solve(H, b, O.Initialization.cold(), cfg)
    assert cold.residual_history[0] == 1.0 and warm.residual_history[0] < cold.residual_history[0]


def test_ap(O):  # test_solvers.cpp:235-331
    H, b = matern_system(O, 22, 25)
    res = O.ap_solve(H, b, O.Initialization.cold(), O.SolverConfig(method=O.AP, block_size=25, tolerance=1e-8))
    assert res.converged and res.iterations == 1
    H1, _ = matern_system(O, 23, 20)
    H2, _ = matern_system(O, 24, 20)
    H = np.zeros((40, 40), order="F")
    H[:20, :20] = H1
    H[20:, 20:] = H2
    b = O.gaussian_vector(25, 40)
    for ordering in (O.AP_GREEDY, O.AP_CYCLIC):
        res = O.ap_solve(H, b, O.Initialization.cold(),
                         O.SolverConfig(method=O.AP, block_size=20, tolerance=1e-10, ap_ordering=ordering))
        assert res.converged and res.iterations <= 2
    H = random_spd(O, 26, 300)
    b = O.gaussian_vector(126, 300)
    res = O.ap_solve(H, b, O.Initialization.cold(), O.SolverConfig(method=O.AP, block_size=100, tolerance=0.01, max_iters=3000))
    assert res.converged and O.relative_residual(H, res.v, b) <= 0.01
    hist = res.residual_history
    assert all(hist[i] <= hist[i - 1] + 1e-12 for i in range(1, len(hist)))
    H, b = matern_system(O, 26, 300, 3, 0.4, 0.4)
    step = O.SolverConfig(method=O.AP, block_size=100, tolerance=0.0)
    jprev = O.quadratic_objective(H, np.zeros(300), b)
    for k in range(1, 31):
        step.max_iters = k
        j = O.quadratic_objective(H, O.ap_solve(H, b, O.Initialization.cold(), step).v, b)
        assert j <= jprev + 1e-12
        jprev = j
    H, b = matern_system(O, 27, 90)
    cfg = O.SolverConfig(method=O.AP, block_size=30, tolerance=1e-6, max_iters=2000)
    a = O.ap_solve(H, b, O.Initialization.cold(), cfg)
    a2 = O.ap_solve(H, b, O.Initialization.cold(), cfg)
    assert np.array_equal(a.v, a2.v)
    Hn = np.eye(4)
    Hn[0, 0] = -1.0
    with pytest.raises(O.NotSpdError):
        O.ap_solve(Hn, O.gaussian_vector(28, 4), O.Initialization.cold(), O.SolverConfig(method=O.AP, block_size=2))


def test_objective_decreases_every_solver(O):  # test_solvers.cpp:333-352
    H, b = matern_system(O, 29, 80, 3, 0.5, 0.6)
    for m in (O.CG, O.SGD, O.AP):
        cfg = O.SolverConfig(method=m, tolerance=0.01, max_iters=5000, learning_rate=0.02, batch_size=20,
                             block_size=25, precond_rank=20, precond_shift=0.36)
        res = O.solve(H, b, O.Initialization.cold(), cfg)
        assert res.iterations >= 1
        assert O.quadratic_objective(H, res.v, b) < O.quadratic_objective(H, np.zeros(80), b)


def test_history_contract(O):  # test_solvers.cpp:354-366
    H, b = matern_system(O, 30, 60, 3, 0.5, 0.5)
    res = O.cg_solve(H, b, O.Initialization.cold(),
                     O.SolverConfig(tolerance=1e-4, max_iters=500, precond_rank=15, precond_shift=0.25))
    assert len(res.residual_history) == res.iterations + 1 and res.residual_history[0] == 1.0
    if res.converged:
        assert res.final_residual() <= 1e-4


@pytest.mark.parametrize("seed", [31, 32, 33, 34, 35])
def test_warm_never_worse_than_cold_plus_one(O, seed):  # test_solvers.cpp:368-395
    H11, H, b1, b = blocked(O, seed, 80, 12, 3, 0.4, 0.5)
    u1 = O.exact_solve(H11, b1)
    for m in (O.CG, O.SGD, O.AP):
        cfg = O.SolverConfig(method=m, tolerance=0.01, max_iters=20000, learning_rate=0.02, batch_size=30,
                             block_size=12, precond_rank=20, precond_shift=0.25)
        cold = O.solve(H, b, O.Initialization.cold(), cfg)
        warm = O.solve(H, b, O.Initialization.warm(u1), cfg)
        assert cold.converged and warm.converged
        assert warm.iterations <= cold.iterations + 1


def test_solve_many(O):  # test_solvers.cpp:397-472
    H, b = matern_system(O, 36, 50, 3, 0.5, 0.5)
    cfg = O.SolverConfig(tolerance=1e-6, precond_rank=10, precond_shift=0.25)
    many = O.solve_many(H, b.reshape(-1, 1), [O.Initialization.cold()], cfg)
    single = O.solve(H, b, O.Initialization.cold(), cfg)
    assert np.array_equal(many[0].v, single.v) and many[0].residual_history == single.residual_history
    B = np.stack([b, b, b], 1)
    for m in (O.CG, O.AP):
        c = O.SolverConfig(method=m, tolerance=1e-6, max_iters=2000, block_size=20, precond_rank=10, precond_shift=0.25)
        r = O.solve_many(H, B, [O.Initialization.cold()] * 3, c)
        assert np.array_equal(r[0].v, r[1].v) and np.array_equal(r[1].v, r[2].v)
    c = O.SolverConfig(method=O.SGD, learning_rate=0.02, batch_size=10, max_iters=100, tolerance=1e-10, seed=9)
    a = O.solve_many(H, B[:, :2], [O.Initialization.cold()] * 2, c)
    a2 = O.solve_many(H, B[:, :2], [O.Initialization.cold()] * 2, c)
    assert np.array_equal(a[0].v, a2[0].v) and np.array_equal(a[1].v, a2[1].v)
    assert not np.array_equal(a[0].v, a[1].v)
    Bm = np.stack([O.gaussian_vector(100 + k, 50) for k in range(100)], 1)
    c = O.SolverConfig(tolerance=0.0, max_iters=5, precond_rank=10, precond_shift=0.25)
    for r in O.solve_many(H, Bm, [O.Initialization.cold()] * 100, c):
        assert r.iterations == 5 and len(r.residual_history) == 6
    with pytest.raises(ValueError):
        O.solve_many(H, B[:, :2], [O.Initialization.cold()], O.SolverConfig())


def test_solver_oracle_acceptance(O):  # verify.cpp:115-173 / acceptance crit. 4
    r = O.Rng(2024)
    worst = 0.0
    for _ in range(2):
        h = O.KernelHyperparams(r.uniform(0.3, 0.8), 1.0, r.uniform(0.4, 0.8))
        X = np.zeros((120, 3), order="F")
        for i in range(120):
            for k in range(3):
                X[i, k] = r.uniform()
        H = O.gram_matrix(X, h)
        b = np.array([r.normal() for _ in range(120)])
        ve = O.exact_solve(H, b)
        en = O.rkhs_distance(H, np.zeros(120), ve)
        for m in (O.CG, O.AP):
            cfg = O.SolverConfig(method=m, tolerance=1e-6, max_iters=200000, batch_size=40, block_size=30,
                                 precond_rank=20, precond_shift=h.noise_scale ** 2)
            res = O.solve(H, b, O.Initialization.cold(), cfg)
            assert res.converged
            worst = max(worst, O.rkhs_distance(H, res.v, ve) / en)
    assert worst <= 1e-4


def test_matrix_free_operator_solves_like_dense(O):
    h = O.KernelHyperparams(0.5, 1.0, 0.3, O.RBF)
    X = O.uniform_inputs(44, 200, 4)
    b = O.gaussian_vector(45, 200)
    H = O.gram_matrix(X, h)
    op = O.Operator(X=X, hyp=h)
    for m in (O.CG, O.AP, O.SGD):
        cfg = O.SolverConfig(method=m, tolerance=1e-5, max_iters=3000, block_size=50, batch_size=50,
                             learning_rate=0.01, precond_rank=20, precond_shift=0.09)
        a = O.solve(H, b, O.Initialization.cold(), cfg)
        c = O.solve(op, b, O.Initialization.cold(), cfg)
        assert abs(a.iterations - c.iterations) <= 1
        np.testing.assert_allclose(a.residual_history[: min(len(a.residual_history), 20)],
                                   c.residual_history[: min(len(a.residual_history), 20)], rtol=1e-8)

"""Oracle pins restated from the reference's kernel tests (proj/tests/test_kernel.cpp) plus
known answers for the RBF extension (parity-unpinned by the reference)."""
import math

import numpy as np
import pytest

SQRT3 = 1.7320508075688772935


def test_matern_point_values(O):  # test_kernel.cpp:13-43
    h = O.KernelHyperparams(1.0, 1.0, 1e-3)
    x = [0.3, -0.2]
    assert O.kernel(x, x, h) == 1.0
    assert O.kernel(x, x, O.KernelHyperparams(0.7, 2.0, 1e-3)) == 4.0
    y = [1.3, -0.2]
    expected = (1.0 + SQRT3) * math.exp(-SQRT3)
    assert O.kernel(x, y, h) == pytest.approx(expected, rel=1e-14)
    assert O.kernel(x, y, h) == pytest.approx(0.483358, rel=1e-6)
    assert O.kernel(x, [100.3, -0.2], O.KernelHyperparams(0.1, 1.0, 1e-3)) < 1e-10
    y = [-0.9, 2.4]
    assert O.kernel(x, y, h) == O.kernel(y, x, h)
    with pytest.raises(ValueError):
        O.kernel(x, [0.0, 0.0, 0.0], h)


def test_matern_strictly_decreasing(O):  # test_kernel.cpp:45-53
    h = O.KernelHyperparams(0.8, 1.3, 1e-3)
    prev = O.kernel_from_distance(h, 0.0)
    for i in range(1, 201):
        cur = O.kernel_from_distance(h, 0.025 * i)
        assert cur < prev
        prev = cur


def test_rbf_known_answers(O):
    h = O.KernelHyperparams(0.5, 1.5, 0.1, O.RBF)
    assert O.kernel_from_distance(h, 0.0) == 2.25
    assert O.kernel_from_distance(h, 0.5) == pytest.approx(2.25 * math.exp(-0.5), rel=1e-15)
    assert O.kernel_from_distance(h, 1.0) == pytest.approx(2.25 * math.exp(-2.0), rel=1e-15)
    assert O.kernel_from_distance(O.KernelHyperparams(0.1, 1.0, 1e-3, O.RBF), 10.0) < 1e-300


def test_gram_single_point(O):  # test_kernel.cpp:55-61
    H = O.gram_matrix(np.array([[0.1, 0.2, 0.3, 0.4]]), O.KernelHyperparams(1.0, 1.0, 0.1))
    assert H.shape == (1, 1) and H[0, 0] == pytest.approx(1.01, rel=1e-14)


@pytest.mark.parametrize("kind", [0, 1])
def test_gram_invariants(O, kind):  # test_kernel.cpp:63-80
    h = O.KernelHyperparams(0.3, 1.0, 0.001, kind)
    H = O.gram_matrix(O.uniform_inputs(5, 50, 8), h)
    assert np.abs(H - H.T).max() == 0.0
    assert np.abs(np.diag(H) - (1.0 + 1e-6)).max() < 1e-12
    assert np.linalg.cholesky(H).diagonal().min() > 0.0


def test_gram_leading_submatrix(O):  # test_kernel.cpp:82-92
    h = O.KernelHyperparams(0.6, 1.2, 0.05)
    X1 = O.uniform_inputs(8, 40, 3)
    X2 = O.uniform_inputs(9, 15, 3)
    full = O.gram_matrix(np.vstack([X1, X2]), h)
    assert np.abs(full[:40, :40] - O.gram_matrix(X1, h)).max() < 1e-12


def test_psd_random_grams(O):  # test_kernel.cpp:94-105
    for seed in (11, 12, 13):
        r = O.Rng(seed)
        n = 50 + r.uniform_index(151)
        dim = 2 + r.uniform_index(7)
        h = O.KernelHyperparams(r.uniform(0.2, 2.0), r.uniform(0.5, 2.0), r.uniform(0.01, 0.5))
        np.linalg.cholesky(O.gram_matrix(O.uniform_inputs(seed + 100, n, dim), h))


def test_cross_kernel(O):  # test_kernel.cpp:107-140
    h = O.KernelHyperparams(0.5, 1.1, 0.2)
    X = O.uniform_inputs(31, 25, 4)
    K = O.cross_kernel(X, X, h)
    expected = O.gram_matrix(X, h) - 0.04 * np.eye(25)
    assert np.abs(K - expected).max() < 1e-12
    a = np.array([[0.4, 0.6]])
    assert O.cross_kernel(a, a, h)[0, 0] == pytest.approx(1.21, rel=1e-14)
    A = O.uniform_inputs(41, 3, 2)
    B = O.uniform_inputs(42, 4, 2)
    K = O.cross_kernel(A, B, h)
    for i in range(3):
        for j in range(4):
            assert K[i, j] == pytest.approx(O.kernel(A[i], B[j], h), rel=1e-12)
    with pytest.raises(ValueError):
        O.cross_kernel(O.uniform_inputs(1, 2, 3), O.uniform_inputs(2, 2, 4), h)


def test_extend_system(O):  # test_kernel.cpp:142-187
    h = O.KernelHyperparams(0.5, 1.0, 0.1)
    X1 = O.uniform_inputs(51, 30, 3)
    X2 = O.uniform_inputs(52, 10, 3)
    H1 = O.gram_matrix(X1, h)
    same = O.extend_assembled(H1, X1, np.zeros((0, 3)), h)
    assert np.array_equal(same, H1)
    H = O.extend_assembled(H1, X1, X2, h)
    assert np.array_equal(H[:30, :30], H1)
    assert np.abs(H - O.gram_matrix(np.vstack([X1, X2]), h)).max() < 1e-12
    with pytest.raises(ValueError):
        O.extend_assembled(H1, X1, O.uniform_inputs(3, 10, 4), h)
    Xa = O.uniform_inputs(61, 1000, 3)
    Xb = O.uniform_inputs(62, 100, 3)
    hb = O.KernelHyperparams(1.5, 1.0, 0.1)
    Hb = O.extend_assembled(O.gram_matrix(Xa, hb), Xa, Xb, hb)
    assert Hb.shape == (1100, 1100) and np.abs(Hb - Hb.T).max() == 0.0


@pytest.mark.parametrize("kind", [0, 1])
def test_matrix_free_matches_dense(O, kind):
    h = O.KernelHyperparams(0.4, 1.2, 0.3, kind)
    X = O.uniform_inputs(77, 333, 5)
    V = np.random.default_rng(3).standard_normal((333, 7))
    H = O.gram_matrix(X, h)
    np.testing.assert_allclose(O.kmatvec(X, h, V), H @ V, rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(O.kmatvec(X, h, V, rows=(100, 200)), (H @ V)[100:200], rtol=1e-13, atol=1e-12)
    Xs = O.uniform_inputs(78, 50, 5)
    np.testing.assert_allclose(O.cross_matvec(Xs, X, h, V), O.cross_kernel(Xs, X, h) @ V, rtol=1e-12, atol=1e-12)


def _grad_case(O):
    hyp = O.KernelHyperparams(0.6, 1.1, 1e-3, O.MATERN32)
    X = O.uniform_inputs(51, 15, 3)
    return hyp, X


def test_oracle_grad_posterior_reference_cases(O):
    """test_sampling.cpp:190-228: zero amplitudes + zero weights give a zero gradient; the
    gradient matches central finite differences of eval_posterior (rel 1e-5); finite at a
    training point."""
    hyp, X = _grad_case(O)
    p = O.sample_prior(hyp, 3, 32, 52)
    p.amplitudes[:] = 0.0
    assert np.abs(O.grad_posterior(hyp, p, X, np.zeros(15), [0.2, 0.4, 0.6])).max() == 0.0
    p = O.sample_prior(hyp, 3, 128, 53)
    w = O.gaussian_vector(54, 15)
    rng = O.Rng(55)
    h = 1e-5
    for _ in range(10):
        x = np.array([rng.uniform() for _ in range(3)])
        g = O.grad_posterior(hyp, p, X, w, x)
        fd = np.zeros(3)
        for d in range(3):
            xp, xm = x.copy(), x.copy()
            xp[d] += h
            xm[d] -= h
            fd[d] = (O.eval_posterior(hyp, p, X, w, xp[None, :])[0] - O.eval_posterior(hyp, p, X, w, xm[None, :])[0]) / (2 * h)
        assert np.linalg.norm(g - fd) / np.linalg.norm(g) < 1e-5
    p = O.sample_prior(hyp, 3, 64, 56)
    assert np.isfinite(O.grad_posterior(hyp, p, X, O.gaussian_vector(57, 15), X[4])).all()


def test_oracle_grad_posterior_rbf_finite_differences(O):
    """RBF extension: the same finite-difference check."""
    hyp = O.KernelHyperparams(0.5, 0.9, 1e-3, O.RBF)
    X = O.uniform_inputs(61, 20, 4)
    p = O.sample_prior(hyp, 4, 64, 62)
    w = O.gaussian_vector(63, 20)
    x = np.array([0.3, 0.7, 0.1, 0.5])
    g = O.grad_posterior(hyp, p, X, w, x)
    h = 1e-5
    fd = np.array([(O.eval_posterior(hyp, p, X, w, (x + h * e)[None, :])[0]
                    - O.eval_posterior(hyp, p, X, w, (x - h * e)[None, :])[0]) / (2 * h) for e in np.eye(4)])
    assert np.linalg.norm(g - fd) / np.linalg.norm(g) < 1e-5


def test_oracle_ascend_peaks_reference_cases(O):
    """test_thompson.cpp:189-232: a single positive representer weight is a radial bump at x0;
    zero steps return the best start; 200 steps at rate 0.01 climb to x0."""
    hyp = O.KernelHyperparams(0.25, 1.0, 1e-3, O.MATERN32)
    x0 = np.array([[0.43, 0.57]])
    silent = O.sample_prior(hyp, 2, 16, 80)
    silent.amplitudes[:] = 0.0
    starts = np.array([[0.35, 0.5], [0.5, 0.62], [0.41, 0.55]])
    w = np.array([2.0])
    vals = [O.eval_posterior(hyp, silent, x0, w, st[None, :])[0] for st in starts]
    bx, bv = O.ascend_peaks(hyp, silent, x0, w, starts, 0, 0.02)
    assert np.array_equal(bx, starts[int(np.argmax(vals))])
    bx, bv = O.ascend_peaks(hyp, silent, x0, w, starts, 200, 0.01)
    peak = O.eval_posterior(hyp, silent, x0, w, x0)[0]
    assert np.linalg.norm(bx - x0[0]) < 1e-2 and bv >= peak - 1e-3 and bv >= max(vals)

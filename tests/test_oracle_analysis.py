"""Oracle pins for the analysis.cpp restatements (mll / optimize_mll / median heuristic),
restating the reference's own cases (proj/tests/test_analysis.cpp:121-215)."""
import numpy as np
import pytest


def test_mll_gradient_matches_central_differences(O):
    """test_analysis.cpp:126-141."""
    X = O.uniform_inputs(19, 50, 3)
    y = O.gaussian_vector(20, 50)
    hyp = O.KernelHyperparams(0.8, 1.1, 0.4)
    res = O.mll(X, y, hyp)
    h = 1e-4
    th = np.log([hyp.lengthscale, hyp.signal_scale, hyp.noise_scale])
    fd = np.zeros(3)
    for k in range(3):
        tp, tm = th.copy(), th.copy()
        tp[k] += h
        tm[k] -= h
        fd[k] = (O.mll(X, y, O.KernelHyperparams(*np.exp(tp))).value
                 - O.mll(X, y, O.KernelHyperparams(*np.exp(tm))).value) / (2 * h)
    assert np.linalg.norm(fd - res.grad) / np.linalg.norm(res.grad) < 1e-5


def test_mll_zero_targets_is_logdet(O):
    """test_analysis.cpp:142-150."""
    X = O.uniform_inputs(19, 50, 3)
    hyp = O.KernelHyperparams(0.8, 1.1, 0.4)
    res = O.mll(X, np.zeros(50), hyp)
    H = O.gram_matrix(X, hyp)
    logdet = 2.0 * np.log(np.diag(np.linalg.cholesky(H))).sum()
    expected = -0.5 * logdet - 0.5 * 50 * np.log(2 * np.pi)
    assert res.value == pytest.approx(expected, rel=1e-12)


def test_mll_matches_eigendecomposition_density(O):
    """test_analysis.cpp:151-164."""
    Xs = O.uniform_inputs(21, 20, 2)
    ys = O.gaussian_vector(22, 20)
    hyp = O.KernelHyperparams(0.8, 1.1, 0.4)
    ev, U = np.linalg.eigh(O.gram_matrix(Xs, hyp))
    w = U.T @ ys
    expected = -0.5 * np.sum(w * w / ev) - 0.5 * np.log(ev).sum() - 0.5 * 20 * np.log(2 * np.pi)
    assert O.mll(Xs, ys, hyp).value == pytest.approx(expected, rel=1e-10)


def test_mll_not_spd_throws(O):
    """test_analysis.cpp:165-170."""
    Xdup = np.array([[0.1], [0.1], [0.1]])
    with pytest.raises(O.NotSpdError):
        O.mll(Xdup, np.ones(3), O.KernelHyperparams(1.0, 1.0, 1e-12))


def test_optimize_mll_zero_steps_and_monotone(O):
    """test_analysis.cpp:174-190."""
    X = O.uniform_inputs(23, 30, 2)
    y = O.gaussian_vector(24, 30)
    init = O.KernelHyperparams(0.7, 1.2, 0.3)
    out = O.optimize_mll(X, y, init, 0, 0.1)
    assert (out.lengthscale, out.signal_scale, out.noise_scale) == (0.7, 1.2, 0.3)
    X = O.uniform_inputs(25, 60, 2)
    y = O.gaussian_vector(26, 60)
    init = O.KernelHyperparams(2.0, 0.5, 0.8)
    out = O.optimize_mll(X, y, init, 40, 0.1)
    assert O.mll(X, y, out).value >= O.mll(X, y, init).value


def test_mll_rbf_extension_gradient(O):
    """RBF analogue (documented extension): gradient against central differences."""
    X = O.uniform_inputs(31, 40, 2)
    y = O.gaussian_vector(32, 40)
    hyp = O.KernelHyperparams(0.5, 0.9, 0.3, O.RBF)
    res = O.mll(X, y, hyp)
    th = np.log([0.5, 0.9, 0.3])
    fd = np.zeros(3)
    for k in range(3):
        tp, tm = th.copy(), th.copy()
        tp[k] += 1e-4
        tm[k] -= 1e-4
        fd[k] = (O.mll(X, y, O.KernelHyperparams(*np.exp(tp), O.RBF)).value
                 - O.mll(X, y, O.KernelHyperparams(*np.exp(tm), O.RBF)).value) / 2e-4
    assert np.linalg.norm(fd - res.grad) / np.linalg.norm(res.grad) < 1e-5


def test_median_heuristic_positive_and_scale_aware(O):
    """test_analysis.cpp:208-215."""
    X = O.uniform_inputs(30, 200, 3)
    base = O.median_heuristic_lengthscale(X)
    assert 0.1 < base < 2.0
    assert O.median_heuristic_lengthscale(10.0 * X) == pytest.approx(10.0 * base, rel=1e-12)

"""GPU parity of the analysis.cpp functions on the device: mll / optimize_mll
against the oracle (itself pinned to test_analysis.cpp's cases in tests/test_oracle_analysis.py)
and the reference's own mll / optimize_mll cases re-run through the C-ABI."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", [0, 1])
def test_mll_matches_oracle(W, O, kind):
    X = O.uniform_inputs(41, 300, 3)
    y = O.gaussian_vector(42, 300)
    ref = O.mll(X, y, O.KernelHyperparams(0.6, 1.3, 0.2, kind))
    got = W.mll(X, y, W.KernelHyperparams(0.6, 1.3, 0.2, kind))
    assert got.value == pytest.approx(ref.value, rel=1e-10, abs=1e-9)
    np.testing.assert_allclose(got.grad, ref.grad, rtol=1e-8, atol=1e-8 * np.abs(ref.grad).max())


def test_mll_reference_cases(W, O):
    """test_analysis.cpp:121-171 through the device: central differences, zero targets, the
    eigendecomposition density, and NotSpdError."""
    X = O.uniform_inputs(19, 50, 3)
    y = O.gaussian_vector(20, 50)
    hyp = W.KernelHyperparams(0.8, 1.1, 0.4)
    res = W.mll(X, y, hyp)
    th = np.log([0.8, 1.1, 0.4])
    fd = np.zeros(3)
    for k in range(3):
        tp, tm = th.copy(), th.copy()
        tp[k] += 1e-4
        tm[k] -= 1e-4
        fd[k] = (W.mll(X, y, W.KernelHyperparams(*np.exp(tp))).value
                 - W.mll(X, y, W.KernelHyperparams(*np.exp(tm))).value) / 2e-4
    assert np.linalg.norm(fd - res.grad) / np.linalg.norm(res.grad) < 1e-5
    H = O.gram_matrix(X, O.KernelHyperparams(0.8, 1.1, 0.4))
    logdet = 2.0 * np.log(np.diag(np.linalg.cholesky(H))).sum()
    assert W.mll(X, np.zeros(50), hyp).value == pytest.approx(-0.5 * logdet - 25 * np.log(2 * np.pi), rel=1e-12)
    Xs = O.uniform_inputs(21, 20, 2)
    ys = O.gaussian_vector(22, 20)
    ev, U = np.linalg.eigh(O.gram_matrix(Xs, O.KernelHyperparams(0.8, 1.1, 0.4)))
    w = U.T @ ys
    expected = -0.5 * np.sum(w * w / ev) - 0.5 * np.log(ev).sum() - 10 * np.log(2 * np.pi)
    assert W.mll(Xs, ys, hyp).value == pytest.approx(expected, rel=1e-10)
    with pytest.raises(W.NotSpdError):
        W.mll(np.array([[0.1], [0.1], [0.1]]), np.ones(3), W.KernelHyperparams(1.0, 1.0, 1e-12))


def test_optimize_mll_matches_oracle_trajectory(W, O):
    """Same Adam trajectory as the oracle (device MLL gradients agree to ~1e-10)."""
    X = O.uniform_inputs(25, 120, 2)
    y = O.gaussian_vector(26, 120)
    ref = O.optimize_mll(X, y, O.KernelHyperparams(2.0, 0.5, 0.8), 25, 0.1)
    got = W.optimize_mll(X, y, W.KernelHyperparams(2.0, 0.5, 0.8), 25, 0.1)
    np.testing.assert_allclose([got.lengthscale, got.signal_scale, got.noise_scale],
                               [ref.lengthscale, ref.signal_scale, ref.noise_scale], rtol=1e-7)


def test_optimize_mll_reference_cases(W, O):
    """test_analysis.cpp:174-205: zero steps return the start, never worse than the start, and
    a known lengthscale (exact GP sample, l = 0.3, n = 500) recovered within a factor of two."""
    X = O.uniform_inputs(23, 30, 2)
    y = O.gaussian_vector(24, 30)
    out = W.optimize_mll(X, y, W.KernelHyperparams(0.7, 1.2, 0.3), 0, 0.1)
    assert (out.lengthscale, out.signal_scale, out.noise_scale) == (0.7, 1.2, 0.3)
    X = O.uniform_inputs(25, 60, 2)
    y = O.gaussian_vector(26, 60)
    init = W.KernelHyperparams(2.0, 0.5, 0.8)
    out = W.optimize_mll(X, y, init, 40, 0.1)
    assert W.mll(X, y, out).value >= W.mll(X, y, init).value
    X = O.uniform_inputs(27, 500, 2)
    K = O.gram_matrix(X, O.KernelHyperparams(0.3, 1.0, 1e-4))
    y = np.linalg.cholesky(K) @ O.gaussian_vector(28, 500) + 0.05 * O.gaussian_vector(29, 500)
    fit = W.optimize_mll(X, y, W.KernelHyperparams(1.0, 1.0, 0.2), 120, 0.15)
    assert 0.15 < fit.lengthscale < 0.6


def test_mll_on_operator_rows(W, O):
    """mll on an existing (grown) operator's rows at its own hyperparameters."""
    X = O.uniform_inputs(51, 400, 4)
    y = O.gaussian_vector(52, 400)
    op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1), X[:300], precision=W.F32_3XTF32)
    op.append_rows(X[300:])
    ref = O.mll(X, y, O.KernelHyperparams(0.5, 1.0, 0.1))
    got = W.mll(op, y)
    assert got.value == pytest.approx(ref.value, rel=1e-10)

"""Device grad_posterior and batched peak ascent against the oracle's
restatements (sampling.cpp:77-87, thompson.cpp:209-258) and the reference's own cases."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", [0, 1])
def test_grad_posterior_matches_oracle(W, O, kind):
    ohyp = O.KernelHyperparams(0.6, 1.1, 1e-3, kind)
    whyp = W.KernelHyperparams(0.6, 1.1, 1e-3, kind)
    X = O.uniform_inputs(51, 400, 3)
    S = 3
    priors_o = [O.sample_prior(ohyp, 3, 128, 53 + s) for s in range(S)]
    priors_w = [W.sample_prior(whyp, 3, 128, 53 + s) for s in range(S)]
    wts = np.column_stack([O.gaussian_vector(60 + s, 400) for s in range(S)])
    pts = O.uniform_inputs(70, 20, 3)
    pts[3] = X[4]  # at a training point: finite (test_sampling.cpp:221-227)
    sidx = np.arange(20) % S
    op = W.KernelOperator(whyp, X, precision=W.F64)
    G = W.grad_posterior(op, priors_w, wts, pts, sidx)
    assert np.isfinite(G).all()
    for i in range(20):
        ref = O.grad_posterior(ohyp, priors_o[sidx[i]], X, wts[:, sidx[i]], pts[i])
        assert np.linalg.norm(G[i] - ref) <= 1e-11 * max(1.0, np.linalg.norm(ref)), i


def test_ascend_peaks_reference_bump(W):
    """test_thompson.cpp:189-232 on the device: zero steps return the best start, 200 steps
    climb to the radial bump's maximizer, never worse than the best start."""
    whyp = W.KernelHyperparams(0.25, 1.0, 1e-3, W.MATERN32)
    x0 = np.array([[0.43, 0.57]])
    silent = W.sample_prior(whyp, 2, 16, 80)
    silent.amplitudes[:] = 0.0
    op = W.KernelOperator(whyp, x0, precision=W.F64)
    starts = np.array([[[0.35, 0.5], [0.5, 0.62], [0.41, 0.55]]])
    w = np.array([[2.0]])
    vals = W.eval_posterior(op, [silent], w, starts[0])[:, 0]
    bx, bv = W.ascend_peaks(op, [silent], w, starts, 0, 0.02)
    assert np.array_equal(bx[0], starts[0, int(np.argmax(vals))])
    bx, bv = W.ascend_peaks(op, [silent], w, starts, 200, 0.01)
    peak = W.eval_posterior(op, [silent], w, x0)[0, 0]
    assert np.linalg.norm(bx[0] - x0[0]) < 1e-2 and bv[0] >= peak - 1e-3 and bv[0] >= vals.max()


def test_ascend_peaks_matches_oracle_batched(W, O):
    """Eight samples x four starts, 60 Adam steps: each sample's best point and value agree
    with the oracle's sequential ascend_peaks."""
    ohyp = O.KernelHyperparams(0.3, 1.0, 1e-3, O.MATERN32)
    whyp = W.KernelHyperparams(0.3, 1.0, 1e-3, W.MATERN32)
    X = O.uniform_inputs(81, 300, 3)
    S, P = 8, 4
    priors_o = [O.sample_prior(ohyp, 3, 256, 90 + s) for s in range(S)]
    priors_w = [W.sample_prior(whyp, 3, 256, 90 + s) for s in range(S)]
    wts = 0.05 * np.column_stack([O.gaussian_vector(100 + s, 300) for s in range(S)])
    starts = O.uniform_inputs(110, S * P, 3).reshape(S, P, 3)
    op = W.KernelOperator(whyp, X, precision=W.F64)
    bx, bv = W.ascend_peaks(op, priors_w, wts, starts, 60, 0.01)
    for s in range(S):
        rx, rv = O.ascend_peaks(ohyp, priors_o[s], X, wts[:, s], starts[s], 60, 0.01)
        assert abs(bv[s] - rv) <= 1e-9 * max(1.0, abs(rv)), s
        assert np.linalg.norm(bx[s] - rx) <= 1e-6, s

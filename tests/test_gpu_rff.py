"""GPU parity of the fused RFF prior evaluation (K7) against the oracle's eval_prior
(sampling.cpp:37-46) and the reference's sampling tests (test_sampling.cpp)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,dim,F,S", [(0, 3, 200, 3), (1, 8, 1024, 2), (0, 16, 2048, 5), (0, 6, 2000, 7)])
def test_rff_eval_vs_oracle(W, O, kind, dim, F, S):
    X = O.uniform_inputs(11 + dim, 777, dim)
    hw = W.KernelHyperparams(0.6, 1.3, 1e-3, kind)
    ho = O.KernelHyperparams(0.6, 1.3, 1e-3, kind)
    op = W.KernelOperator(hw, X)
    priors = [W.sample_prior(hw, dim, F, W.derive_seed(5, p)) for p in range(S)]
    got = W.rff_eval(op, priors)
    Xs = O.uniform_inputs(99, 123, dim)
    got_s = W.rff_eval(op, priors, Xs)
    for p in range(S):
        po = O.sample_prior(ho, dim, F, O.derive_seed(5, p))
        ref = O.eval_prior(po, X)
        np.testing.assert_allclose(got[:, p], ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))
        np.testing.assert_allclose(got_s[:, p], O.eval_prior(po, Xs), rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))


def test_zero_frequency_constant_and_zero_amplitudes(W):  # test_sampling.cpp:95-118
    hw = W.KernelHyperparams(0.5, 1.3, 1e-3)
    X = np.random.default_rng(3).random((15, 2))
    op = W.KernelOperator(hw, X)
    p = W.RffPrior(np.zeros((1, 2), order="F"), np.zeros(1), np.full(1, 0.8), 1.3)
    vals = W.rff_eval(op, [p])[:, 0]
    assert np.abs(vals - 1.3 * np.sqrt(2.0) * 0.8).max() < 1e-14
    q = W.sample_prior(hw, 2, 50, 1)
    q.amplitudes[:] = 0.0
    assert np.abs(W.rff_eval(op, [q])).max() == 0.0


def test_build_sample_rhs_vs_oracle(W, O):
    X = O.uniform_inputs(22, 500, 3)
    op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 1e-3), X)
    pw = W.sample_prior(W.KernelHyperparams(0.5, 1.0, 1e-3), 3, 256, 21)
    po = O.sample_prior(O.KernelHyperparams(0.5, 1.0, 1e-3), 3, 256, 21)
    a = W.build_sample_rhs(op, pw, 0.05, 1)
    b = O.build_sample_rhs(po, X, 0.05, 1)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)

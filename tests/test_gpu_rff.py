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


def test_rff_eval_fast_close_to_fp64(W):
    """wgp_rff_eval_fast (fp32 phases, reduced MUFU cos) tracks the fp64 kernel to ~1e-6 of the
    prior's scale at BO-like sizes (F = 2000, phases up to |w.x| ~ 30)."""
    import numpy as np
    rng = np.random.default_rng(2)
    for kind, ls, d in ((0, 0.3, 4), (1, 0.5, 6)):
        hyp = W.KernelHyperparams(ls, 1.0, 1e-3, kind)
        X = rng.random((500, d))
        op = W.KernelOperator(hyp, X, precision=W.F32_3XTF32)
        priors = [W.sample_prior(hyp, d, 2000, W.derive_seed(9, s)) for s in range(5)]
        Xc = rng.random((20000, d))
        ref = W.rff_eval(op, priors, Xc)
        got = W.rff_eval(op, priors, Xc, fast=True)
        assert np.abs(got - ref).max() <= 2e-5 * np.abs(ref).max()


def test_bo_candidates_fast_path(W):
    """The BO loop's candidate evaluation on the tensor-core twin + fp32 RFF agrees with the
    fp64 evaluation (same solved weights) and picks the same argmax for nearly every sample."""
    import numpy as np
    from paper_2511_16340_b200 import configs as Cfg
    X0 = Cfg.uniform_rows_fast(3, 1500, 3)
    y0 = np.sin(5 * X0[:, 0]) + X0[:, 1]
    hyp = W.KernelHyperparams(0.3, 1.0, 1e-3, W.MATERN32)
    st = Cfg.growth_state(X0, y0, hyp, 16, 2000, 3, W.F64)
    st.solve_round(W.SolverConfig(tolerance=1e-2, max_iters=5, precond_rank=100, precond_shift=1e-6), warm=True)
    Xc = Cfg.uniform_rows_fast(4, 30000, 3)
    ref = Cfg.posterior_at(st, Xc)
    st.op_fast = W.KernelOperator(hyp, X0, precision=W.F32_3XTF32)
    got = Cfg.posterior_at(st, Xc)
    assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()
    assert np.mean(np.argmax(got, 0) == np.argmax(ref, 0)) >= 0.9

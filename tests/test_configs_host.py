"""CPU checks of the configuration drivers' host logic (no GPU): RNG-derived inputs and
the bump objective."""
import numpy as np


def test_uniform_rows_fast_matches_reference_stream(O):
    from paper_2511_16340_b200 import configs as Cfg
    for seed in (0, 7, 2**63 + 5):
        a = Cfg.uniform_rows_fast(seed, 37, 5)
        b = O.uniform_inputs(seed, 37, 5)  # row-major fill order, testutil.hpp:9-16
        assert np.array_equal(a, b)


def test_init_weights_mirror(W):
    v = W.init_weights(W.Initialization.warm([1.0, 2.0]), 2, 1)
    assert list(v) == [1.0, 2.0, 0.0]
    assert not W.init_weights(W.Initialization.cold(), 3, 2).any()


def test_bump_objective_deterministic():
    from paper_2511_16340_b200 import configs as Cfg
    a = Cfg.BumpObjective.make(3, 11)
    b = Cfg.BumpObjective.make(3, 11)
    X = np.random.default_rng(0).random((10, 3))
    assert np.array_equal(a.value(X), b.value(X))
    assert a.centers.shape == (20, 3) and (a.widths >= 0.05).all() and (a.amps >= 0.5).all()
    assert np.array_equal(a.observe(X), b.observe(X))


def test_solve_many_return_status_raises_not_spd(W, monkeypatch):
    """with return_status=True only DIVERGED is a per-column outcome; a NOT_SPD
    solve wrote no outputs and must raise (solve_best_effort catches DivergenceError only,
    thompson.cpp:299-317).  The library call is stubbed: no GPU needed."""
    import pytest

    class FakeLib:
        def wgp_solve_many(self, *a):
            return W.NOT_SPD

        def wgp_last_error(self):
            return b"cg_solve: non-positive curvature encountered"

    class FakeOp:
        n = 4
        _h = None

    cfg = W.SolverConfig.__new__(W.SolverConfig)  # a ctypes struct: no library call
    cfg.max_iters = 10
    monkeypatch.setattr(W, "lib", lambda: FakeLib())
    B = np.ones((4, 2), order="F")
    with pytest.raises(W.NotSpdError):
        W.solve_many(FakeOp(), B, [W.Initialization.cold()] * 2, cfg, return_status=True)

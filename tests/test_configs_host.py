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

"""The C oracle against outputs of the REFERENCE's own solver code (tests/golden/ref_golden.json,
produced by tests/golden/make_ref_golden.py from the reference's kernel.cpp / solvers.cpp /
sampling.cpp compiled unchanged into oracle/_ref/libwarmgp_ref.so).  Inputs are regenerated
from the recorded seeds through the reference-pinned RNG helpers.

Tolerances: the reference was compiled against an eager Eigen stand-in with plain sequential
reductions, the oracle sums in its own order, so dense results agree to rounding (1e-12
relative); CG is chaotic in the iterate, so the solver checks are: iteration
counts identical (SGD, AP) or within one (CG, at ~40 iterations), identical convergence
flags, histories to 1e-5 relative over the first 10 entries -- and over the whole run for
SGD and AP, which follow one RNG stream / a deterministic block order and are not chaotic --
and solutions to the solver's own accuracy."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_golden.json")))["cases"]


def hyp(h):
    return O.KernelHyperparams(h[0], h[1], h[2], O.MATERN32)


def test_gram_cross_and_kernel_values():
    c = GOLD["gram"]
    X = O.uniform_inputs(c["seed"], c["n"], c["d"])
    H = O.gram_matrix(X, hyp(c["hyp"]))
    ref = np.asarray(c["H"]).reshape(c["n"], c["n"], order="F")
    np.testing.assert_allclose(H, ref, rtol=1e-12, atol=1e-14)
    assert np.array_equal(H, H.T) and np.array_equal(ref, ref.T)
    k = GOLD["cross_kernel"]
    Xs = O.uniform_inputs(k["seed_star"], k["m"], c["d"])
    np.testing.assert_allclose(O.cross_kernel(Xs, X, hyp(c["hyp"])),
                               np.asarray(k["K"]).reshape(k["m"], c["n"], order="F"), rtol=1e-12, atol=1e-14)
    m = GOLD["matern32_from_distance"]
    for r, kv in zip(m["r"], m["k"]):
        assert O.kernel_from_distance(hyp(m["hyp"]), r) == pytest.approx(kv, rel=1e-15, abs=0)


def test_extend_system_assembled():
    c = GOLD["extend_system"]
    X1, X2 = O.uniform_inputs(c["seeds"][0], c["n1"], 3), O.uniform_inputs(c["seeds"][1], c["n2"], 3)
    h = hyp(c["hyp"])
    H = O.extend_assembled(O.gram_matrix(X1, h), X1, X2, h)
    n = c["n1"] + c["n2"]
    np.testing.assert_allclose(H, np.asarray(c["H"]).reshape(n, n, order="F"), rtol=1e-12, atol=1e-14)


def test_pivoted_cholesky_and_preconditioner():
    c = GOLD["pivoted_cholesky"]
    X = O.uniform_inputs(c["seed"], c["n"], 3)
    H = O.gram_matrix(X, hyp(c["hyp"]))
    L = O.pivoted_cholesky(H, c["rank"])
    assert L.shape[1] == c["achieved"]
    np.testing.assert_allclose(L, np.asarray(c["L"]).reshape(c["n"], c["achieved"], order="F"), rtol=1e-10, atol=1e-12)
    p = GOLD["precond_apply"]
    r = O.gaussian_vector(p["seed_r"], c["n"])
    for mode, z in p["z_by_mode"].items():
        pre = O.CgPreconditioner.from_matrix(H, p["rank"], p["shift"], int(mode))
        np.testing.assert_allclose(pre.apply(r), z, rtol=1e-9, atol=1e-12)


def _system():
    s = GOLD["solvers"]
    X = O.uniform_inputs(s["seed_X"], s["n"], s["d"])
    h = hyp(s["hyp"])
    H = O.gram_matrix(X, h)
    b = O.gaussian_vector(s["seed_b"], s["n"])
    u1 = np.linalg.solve(O.gram_matrix(X[: s["warm_rows"]], h), b[: s["warm_rows"]])
    return H, b, u1


def _check_run(got, ref, name, count_tol=0):
    """count_tol: CG counts may differ by one -- the residual crosses the tolerance within
    one step under rounding-level perturbations of the iterate (reduction order)."""
    assert abs(got.iterations - ref["iterations"]) <= count_tol, (name, got.iterations, ref["iterations"])
    assert got.converged == ref["converged"], name
    k = min(10, len(ref["history"]), len(got.residual_history))
    np.testing.assert_allclose(got.residual_history[:k], ref["history"][:k], rtol=1e-5, err_msg=name)
    assert len(got.residual_history) == got.iterations + 1, name
    # the solution agrees to the solve's own accuracy (the last residuals of a converged CG
    # differ by rounding-driven amounts below the tolerance)
    v, vr = np.asarray(got.v), np.asarray(ref["v"])
    assert np.linalg.norm(v - vr) <= 1e-4 * np.linalg.norm(vr) + 1e-12, name


@pytest.mark.parametrize("name", ["cg", "cg_noise_only", "cg_rank0", "sgd", "sgd_block", "ap_greedy", "ap_cyclic"])
@pytest.mark.parametrize("start", ["cold", "warm"])
def test_solvers_match_reference(name, start):
    H, b, u1 = _system()
    run = GOLD["solvers"]["runs"][name]
    cfg = O.SolverConfig(**run["cfg"])
    init = O.Initialization.cold() if start == "cold" else O.Initialization.warm(u1)
    got = O.solve(H, b, init, cfg)
    _check_run(got, run[start], f"{name}/{start}", count_tol=1 if name.startswith("cg") else 0)
    if name.startswith(("sgd", "ap")):  # one RNG stream / deterministic block order: not chaotic
        np.testing.assert_allclose(got.residual_history, run[start]["history"], rtol=1e-8)


@pytest.mark.parametrize("name", ["cg", "sgd", "ap"])
def test_solve_many_matches_reference(name):
    H, _, _ = _system()
    c = GOLD["solve_many"]
    B = np.column_stack([O.gaussian_vector(s, H.shape[0]) for s in c["seeds_b"]])
    run = c["runs"][name]
    res = O.solve_many(H, B, [O.Initialization.cold()] * 3, O.SolverConfig(**run["cfg"]))
    V = np.asarray(run["V"]).reshape(H.shape[0], 3, order="F")
    for i, r in enumerate(res):
        _check_run(r, {"iterations": run["iterations"][i], "converged": run["converged"][i],
                       "history": run["history"][i], "v": V[:, i]}, f"{name}[{i}]",
                   count_tol=1 if name == "cg" else 0)


def test_error_semantics_match_reference():
    H, b, _ = _system()
    z = GOLD["zero_rhs"]
    got = O.solve(H, np.zeros(H.shape[0]), O.Initialization.cold(), O.SolverConfig(method=0, tolerance=1e-6, max_iters=50))
    assert z["status"] == 0 and got.iterations == z["iterations"] == 0
    assert got.residual_history == z["history"] == [0.0] and got.converged and z["converged"]
    d = GOLD["sgd_divergence"]
    assert d["status"] == 2
    with pytest.raises(O.DivergenceError) as e:
        O.solve(H, b, O.Initialization.cold(), O.SolverConfig(**d["cfg"]))
    assert e.value.iterations == d["iterations"]
    Hbad = np.diag(np.concatenate([np.ones(5), -np.ones(5)]))
    for key, kw in (("cg_not_spd", dict(method=0, tolerance=1e-10, max_iters=50, precond_rank=0)),
                    ("ap_not_spd", dict(method=2, tolerance=1e-10, max_iters=50, block_size=5))):
        assert GOLD[key]["status"] == 1
        with pytest.raises(O.NotSpdError):
            O.solve(Hbad, np.ones(10), O.Initialization.cold(), O.SolverConfig(**kw))
    rr = GOLD["relative_residual"]
    v = np.asarray(GOLD["solvers"]["runs"]["cg"]["cold"]["v"])
    assert O.relative_residual(H, v, b) == pytest.approx(rr["value"], rel=1e-9)


def test_sampling_matches_reference():
    s = GOLD["sampling"]
    h = hyp(s["hyp"])
    p = O.sample_prior(h, s["dim"], s["F"], s["seed"])
    F, d = s["F"], s["dim"]
    np.testing.assert_array_equal(p.frequencies, np.asarray(s["frequencies"]).reshape(F, d, order="F"))
    np.testing.assert_array_equal(p.phases, s["phases"])
    np.testing.assert_array_equal(p.amplitudes, s["amplitudes"])
    Xq = O.uniform_inputs(s["seed_Xq"], 10, d)
    np.testing.assert_allclose(O.eval_prior(p, Xq), s["eval_prior"], rtol=1e-12, atol=1e-13)
    Xt = O.uniform_inputs(s["seed_Xt"], 20, d)
    np.testing.assert_allclose(O.build_sample_rhs(p, Xt, s["rhs_noise"], s["rhs_seed"]), s["build_sample_rhs"],
                               rtol=1e-12, atol=1e-13)
    w = O.gaussian_vector(s["seed_w"], 20)
    np.testing.assert_allclose(O.eval_posterior(h, p, Xt, w, Xq), s["eval_posterior"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(O.grad_posterior(h, p, Xt, w, Xq[s["grad_posterior_at_row"]]), s["grad_posterior"],
                               rtol=1e-11, atol=1e-13)

"""Generate tests/golden/ref_golden.json from the REFERENCE's own solver code.

oracle/_ref/libwarmgp_ref.so is the reference's kernel.cpp, solvers.cpp and sampling.cpp
compiled unchanged from /root/reference (oracle/Makefile `ref`, against the eager Eigen
stand-in oracle/eigen_shim).  This script runs it on seeded inputs (the reference Rng streams,
regenerated in the tests from the same seeds through oracle.uniform_inputs /
gaussian_vector, which are pinned bit-for-bit to the reference rng.hpp) and freezes the
outputs: kernel matrices, the pivoted Cholesky factor, preconditioner applications, CG /
SGD / AP iteration counts, residual histories and solutions, solve_many, the error
semantics (zero RHS, divergence, non-SPD), RFF priors and posterior evaluations.

Run in the build container (the reference tree is mounted only there):
    make -C oracle ref && python tests/golden/make_ref_golden.py
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402  (input generation: reference-pinned RNG streams)

LIB = os.path.join(ROOT, "oracle", "_ref", "libwarmgp_ref.so")
OUT = os.path.join(ROOT, "tests", "golden", "ref_golden.json")
P = C.c_void_p
I64 = C.c_int64
D = C.c_double


class RefCfg(C.Structure):
    _fields_ = [("method", C.c_int), ("tolerance", D), ("max_iters", C.c_int), ("learning_rate", D),
                ("momentum", D), ("batch_size", I64), ("sgd_scaling", C.c_int), ("block_size", I64),
                ("ap_ordering", C.c_int), ("precond_rank", I64), ("precond_shift", D),
                ("precond_shift_mode", C.c_int), ("seed", C.c_uint64)]


class RefResult(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("converged", C.c_int), ("hist_len", I64)]


DEFAULTS = dict(method=0, tolerance=1e-2, max_iters=1000, learning_rate=0.3, momentum=0.9, batch_size=100,
                sgd_scaling=0, block_size=100, ap_ordering=0, precond_rank=100, precond_shift=1e-6,
                precond_shift_mode=0, seed=0)  # solvers.hpp:27-48


def cfg(**kw):
    d = dict(DEFAULTS)
    d.update(kw)
    return RefCfg(**d), d


def f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def ptr(a):
    return None if a is None else a.ctypes.data_as(P)


L = C.CDLL(LIB)
L.ref_matern32_from_distance.restype = D
L.ref_matern32_from_distance.argtypes = [D, D, D, D]
L.ref_pivoted_cholesky.restype = I64
L.ref_relative_residual.restype = D
for name in ("ref_gram_matrix", "ref_cross_kernel", "ref_pivoted_cholesky", "ref_precond_apply", "ref_solve",
             "ref_solve_many", "ref_cg_solve_with", "ref_relative_residual", "ref_sample_prior", "ref_eval_prior",
             "ref_build_sample_rhs", "ref_eval_posterior", "ref_grad_posterior", "ref_extend_system"):
    getattr(L, name).argtypes = None  # variadic-style calls with explicit ctypes values below


def gram(X, ls, sf, sn):
    n, d = X.shape
    H = np.zeros((n, n), order="F")
    L.ref_gram_matrix(ptr(f(X)), I64(n), I64(d), D(ls), D(sf), D(sn), ptr(H))
    return H


def solve(H, b, u1, c):
    n = H.shape[0]
    v = np.zeros(n)
    hist = np.zeros(c.max_iters + 2)
    r = RefResult()
    u = None if u1 is None else f(u1)
    L.ref_solve(ptr(f(H)), I64(n), ptr(f(b)), ptr(u), I64(0 if u is None else u.size), C.byref(c), ptr(v),
                ptr(hist), I64(hist.size), C.byref(r))
    return {"status": r.status, "iterations": r.iterations, "converged": bool(r.converged),
            "history": hist[: r.hist_len].tolist() if r.status == 0 else [], "v": v.tolist() if r.status == 0 else []}


def main():
    g = {"generator": "tests/golden/make_ref_golden.py", "library": "oracle/_ref/libwarmgp_ref.so "
         "(reference kernel.cpp + solvers.cpp + sampling.cpp, unchanged, eager Eigen stand-in)",
         "inputs": "X = oracle.uniform_inputs(seed, n, d); b = oracle.gaussian_vector(seed', n) "
                   "(reference Rng streams)", "cases": {}}
    cases = g["cases"]

    # kernel matrices (kernel.cpp:17-89)
    X = O.uniform_inputs(101, 40, 3)
    cases["gram"] = {"seed": 101, "n": 40, "d": 3, "hyp": [0.7, 1.3, 0.2], "H": gram(X, 0.7, 1.3, 0.2).ravel("F").tolist()}
    Xs = O.uniform_inputs(102, 7, 3)
    K = np.zeros((7, 40), order="F")
    L.ref_cross_kernel(ptr(f(Xs)), I64(7), ptr(f(X)), I64(40), I64(3), D(0.7), D(1.3), D(0.2), ptr(K))
    cases["cross_kernel"] = {"seed_star": 102, "m": 7, "K": K.ravel("F").tolist()}
    cases["matern32_from_distance"] = {"hyp": [0.7, 1.3, 0.2], "r": [0.0, 0.1, 0.7, 2.5, -0.3],
                                       "k": [L.ref_matern32_from_distance(r, 0.7, 1.3, 0.2)
                                             for r in (0.0, 0.1, 0.7, 2.5, -0.3)]}
    X1, X2 = O.uniform_inputs(103, 30, 3), O.uniform_inputs(104, 10, 3)
    Hx = np.zeros((40, 40), order="F")
    L.ref_extend_system(ptr(f(X1)), I64(30), ptr(f(X2)), I64(10), I64(3), D(0.5), D(1.0), D(0.1), ptr(Hx))
    cases["extend_system"] = {"seeds": [103, 104], "n1": 30, "n2": 10, "hyp": [0.5, 1.0, 0.1],
                              "H": Hx.ravel("F").tolist()}

    # pivoted Cholesky + preconditioner (solvers.cpp:72-140)
    Xp = O.uniform_inputs(105, 60, 3)
    Hp = gram(Xp, 0.5, 1.0, 0.1)
    Lf = np.zeros((60, 12), order="F")
    k = L.ref_pivoted_cholesky(ptr(f(Hp)), I64(60), I64(12), ptr(Lf))
    r = O.gaussian_vector(106, 60)
    zs = {}
    for mode in (0, 1):
        z = np.zeros(60)
        L.ref_precond_apply(ptr(f(Hp)), I64(60), I64(12), D(0.01), C.c_int(mode), ptr(f(r)), ptr(z))
        zs[str(mode)] = z.tolist()
    cases["pivoted_cholesky"] = {"seed": 105, "n": 60, "hyp": [0.5, 1.0, 0.1], "rank": 12, "achieved": int(k),
                                 "L": Lf[:, :k].ravel("F").tolist()}
    cases["precond_apply"] = {"seed_r": 106, "rank": 12, "shift": 0.01, "z_by_mode": zs}

    # solvers (solvers.cpp:142-309): one system, cold and warm, each method
    n, d, hy = 200, 4, [0.6, 1.0, 0.3]
    Xs_ = O.uniform_inputs(107, n, d)
    H = gram(Xs_, *hy)
    b = O.gaussian_vector(108, n)
    H1 = gram(Xs_[:190], *hy)
    u1 = np.linalg.solve(H1, b[:190])
    solves = {}
    for name, kw in (("cg", dict(method=0, tolerance=1e-9, max_iters=500, precond_rank=20, precond_shift=0.09)),
                     ("cg_noise_only", dict(method=0, tolerance=1e-9, max_iters=500, precond_rank=20,
                                            precond_shift=0.09, precond_shift_mode=1)),
                     ("cg_rank0", dict(method=0, tolerance=1e-8, max_iters=500, precond_rank=0)),
                     ("sgd", dict(method=1, tolerance=1e-3, max_iters=3000, learning_rate=0.004, batch_size=40, seed=77)),
                     ("sgd_block", dict(method=1, tolerance=1e-3, max_iters=3000, learning_rate=0.05, batch_size=40,
                                        sgd_scaling=1, seed=78)),
                     ("ap_greedy", dict(method=2, tolerance=1e-6, max_iters=3000, block_size=40)),
                     ("ap_cyclic", dict(method=2, tolerance=1e-6, max_iters=3000, block_size=40, ap_ordering=1))):
        c, dd = cfg(**kw)
        solves[name] = {"cfg": dd, "cold": solve(H, b, None, c), "warm": solve(H, b, u1, c)}
    cases["solvers"] = {"seed_X": 107, "seed_b": 108, "n": n, "d": d, "hyp": hy, "warm_rows": 190,
                        "warm_u1": "numpy.linalg.solve(gram(X[:190]), b[:190])", "runs": solves}

    # solve_many (solvers.cpp:311-354): shared preconditioner (CG), per-column seeds (SGD)
    B = np.column_stack([O.gaussian_vector(109 + c, n) for c in range(3)])
    many = {}
    for name, kw in (("cg", dict(method=0, tolerance=1e-8, max_iters=500, precond_rank=15, precond_shift=0.09)),
                     ("sgd", dict(method=1, tolerance=1e-3, max_iters=3000, learning_rate=0.004, batch_size=40, seed=5)),
                     ("ap", dict(method=2, tolerance=1e-6, max_iters=3000, block_size=50))):
        c, dd = cfg(**kw)
        V = np.zeros((n, 3), order="F")
        hist = np.zeros((c.max_iters + 2, 3), order="F")
        res = (RefResult * 3)()
        L.ref_solve_many(ptr(f(H)), I64(n), ptr(f(B)), I64(3), None, I64(0), C.byref(c), ptr(V), ptr(hist),
                         I64(hist.shape[0]), res)
        many[name] = {"cfg": dd, "status": res[0].status,
                      "iterations": [res[i].iterations for i in range(3)],
                      "converged": [bool(res[i].converged) for i in range(3)],
                      "history": [hist[: res[i].hist_len, i].tolist() for i in range(3)],
                      "V": V.ravel("F").tolist()}
    cases["solve_many"] = {"seeds_b": [109, 110, 111], "runs": many}

    # error semantics
    c, _ = cfg(method=0, tolerance=1e-6, max_iters=50)
    cases["zero_rhs"] = solve(H, np.zeros(n), None, c)
    c, dd = cfg(method=1, tolerance=1e-6, max_iters=200, learning_rate=5.0, batch_size=40, seed=3)
    cases["sgd_divergence"] = {"cfg": dd, **solve(H, b, None, c)}
    Hbad = np.diag(np.concatenate([np.ones(5), -np.ones(5)]))
    c, dd = cfg(method=0, tolerance=1e-10, max_iters=50, precond_rank=0)
    cases["cg_not_spd"] = {"H": "diag(1 x5, -1 x5)", "b": "ones(10)", **solve(Hbad, np.ones(10), None, c)}
    c, dd = cfg(method=2, tolerance=1e-10, max_iters=50, block_size=5)
    cases["ap_not_spd"] = {"H": "diag(1 x5, -1 x5)", "b": "ones(10)", **solve(Hbad, np.ones(10), None, c)}
    vv = np.asarray(solves["cg"]["cold"]["v"])
    cases["relative_residual"] = {"of": "solvers.runs.cg.cold.v",
                                  "value": L.ref_relative_residual(ptr(f(H)), I64(n), ptr(f(vv)), ptr(f(b)))}

    # sampling (sampling.cpp:14-87)
    F, dd_ = 32, 3
    freq = np.zeros((F, dd_), order="F")
    ph, am = np.zeros(F), np.zeros(F)
    L.ref_sample_prior(D(0.5), D(1.2), D(0.1), I64(dd_), I64(F), C.c_uint64(9), ptr(freq), ptr(ph), ptr(am))
    Xq = O.uniform_inputs(112, 10, dd_)
    ev = np.zeros(10)
    L.ref_eval_prior(ptr(freq), ptr(ph), ptr(am), D(1.2), I64(F), I64(dd_), ptr(f(Xq)), I64(10), ptr(ev))
    Xt = O.uniform_inputs(113, 20, dd_)
    rhs = np.zeros(20)
    L.ref_build_sample_rhs(ptr(freq), ptr(ph), ptr(am), D(1.2), I64(F), I64(dd_), ptr(f(Xt)), I64(20), D(0.1),
                           C.c_uint64(14), ptr(rhs))
    w = O.gaussian_vector(114, 20)
    post = np.zeros(10)
    L.ref_eval_posterior(ptr(freq), ptr(ph), ptr(am), D(1.2), I64(F), I64(dd_), ptr(f(Xt)), I64(20), ptr(f(w)),
                         D(0.5), D(0.1), ptr(f(Xq)), I64(10), ptr(post))
    grad = np.zeros(dd_)
    L.ref_grad_posterior(ptr(freq), ptr(ph), ptr(am), D(1.2), I64(F), I64(dd_), ptr(f(Xt)), I64(20), ptr(f(w)),
                         D(0.5), D(0.1), ptr(f(Xq[3])), ptr(grad))
    cases["sampling"] = {"hyp": [0.5, 1.2, 0.1], "dim": dd_, "F": F, "seed": 9,
                         "frequencies": freq.ravel("F").tolist(), "phases": ph.tolist(), "amplitudes": am.tolist(),
                         "seed_Xq": 112, "eval_prior": ev.tolist(), "seed_Xt": 113, "rhs_noise": 0.1,
                         "rhs_seed": 14, "build_sample_rhs": rhs.tolist(), "seed_w": 114,
                         "eval_posterior": post.tolist(), "grad_posterior_at_row": 3,
                         "grad_posterior": grad.tolist()}

    with open(OUT, "w") as fh:
        json.dump(g, fh, separators=(",", ":"))
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e3:.0f} kB)")
    for name, rec in solves.items():
        print(f"  {name}: cold {rec['cold']['iterations']} it (status {rec['cold']['status']}), "
              f"warm {rec['warm']['iterations']} it")
    for name, rec in many.items():
        print(f"  solve_many {name}: {rec['iterations']}")
    print("  sgd divergence:", cases["sgd_divergence"]["status"], cases["sgd_divergence"]["iterations"],
          " cg not spd:", cases["cg_not_spd"]["status"], " ap not spd:", cases["ap_not_spd"]["status"])


if __name__ == "__main__":
    main()

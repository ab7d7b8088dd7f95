"""Regenerates the committed golden fixtures in tests/golden/.

* rng_golden.json -- streams from the REFERENCE's own rng.hpp, compiled unchanged by
  `make -C oracle ref` (oracle/_ref/rng_golden).  Needs /root/reference (this container).
* kmatvec_*.npz / cg_*.npz -- seeded inputs and oracle outputs at reduced sizes of the
  BASELINE configs; the GPU parity tests compare the CUDA path against these.

Run: python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def rng_golden():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "rng_golden")], check=True,
                         capture_output=True, text=True).stdout
    data = json.loads(out)
    data["source"] = "/root/reference/proj/core/include/warmgp/rng.hpp via oracle/rng_golden_main.cpp"
    with open(os.path.join(HERE, "rng_golden.json"), "w") as f:
        json.dump(data, f, indent=1)


KM_CASES = {
    # name: (kind, lengthscale, signal, noise_scale, n, d, s, input kind, seed)
    "c1_rbf_f64": (O.RBF, 0.5, 1.0, 0.1, 300, 8, 1, "uniform", 11),
    "c3_matern_d16": (O.MATERN32, 0.8, 1.0, 1e-3 ** 0.5, 517, 16, 64, "normal", 12),
    "c4_rbf_d8": (O.RBF, 0.5, 1.0, 0.1, 450, 8, 32, "uniform", 13),
    "c5_matern_d6_s129": (O.MATERN32, 0.3, 1.0, 1e-3, 200, 6, 129, "uniform", 14),
}


def inputs(kind, n, d, seed):
    if kind == "uniform":
        return O.uniform_inputs(seed, n, d)
    r = O.Rng(seed)
    X = np.zeros((n, d), order="F")
    for i in range(n):
        for k in range(d):
            X[i, k] = r.normal()
    return X


def kmatvec_golden():
    for name, (kind, ls, sf, sn, n, d, s, ik, seed) in KM_CASES.items():
        h = O.KernelHyperparams(ls, sf, sn, kind)
        X = inputs(ik, n, d, seed)
        V = np.asfortranarray(np.stack([O.gaussian_vector(O.derive_seed(seed, 100 + c), n) for c in range(s)], 1))
        H = O.gram_matrix(X, h)
        Y = H @ V
        np.savez_compressed(os.path.join(HERE, f"kmatvec_{name}.npz"), X=X, V=V, Y=Y,
                            hyp=np.array([kind, ls, sf, sn]))


def cg_golden():
    # Config-1 protocol at reduced size (bench_regression.cpp:139-197): X uniform^8,
    # RBF l=0.5, s=1, sigma_n^2=1e-2, y = RFF prior (1024 features) + noise, exact u1 on the
    # first n1 rows, CG warm vs cold to 1e-6 (precond rank 100, calibrated, shift sigma_n^2).
    n1, n = 380, 400
    h = O.KernelHyperparams(0.5, 1.0, 0.1, O.RBF)
    X = O.uniform_inputs(O.derive_seed(1, 1), n, 8)
    prior = O.sample_prior(h, 8, 1024, O.derive_seed(1, 7))
    y = O.build_sample_rhs(prior, X, 0.1, O.derive_seed(1, 8))
    H1 = O.gram_matrix(X[:n1], h)
    u1 = O.exact_solve(H1, y[:n1])
    H = O.gram_matrix(X, h)
    cfg = O.SolverConfig(tolerance=1e-6, precond_rank=100, precond_shift=0.01)
    cold = O.cg_solve(H, y, O.Initialization.cold(), cfg)
    warm = O.cg_solve(H, y, O.Initialization.warm(u1), cfg)
    np.savez_compressed(os.path.join(HERE, "cg_c1_reduced.npz"), X=X, y=y, u1=u1,
                        cold_v=cold.v, cold_hist=np.array(cold.residual_history),
                        warm_v=warm.v, warm_hist=np.array(warm.residual_history),
                        hyp=np.array([O.RBF, 0.5, 1.0, 0.1]))


if __name__ == "__main__":
    rng_golden()
    kmatvec_golden()
    cg_golden()
    print("golden fixtures written to", HERE)

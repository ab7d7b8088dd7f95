"""CPU-side checks of the product boundary: libwarmgp_b200.so loads (no GPU needed to
load), exports every symbol include/warmgp_capi.h declares, and its host-only entry
points (shard partition, defaults, RNG) behave like the reference."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "warmgp_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wgp_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_all_exported(W):
    L = W.lib()
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(W.EXPORTS)


def test_abi_version_and_defaults(W):
    assert W.lib().wgp_abi_version() == 2
    c = W.SolverConfig()  # solvers.hpp:27-48
    assert (c.method, c.tolerance, c.max_iters, c.learning_rate, c.momentum) == (W.CG, 1e-2, 1000, 0.3, 0.9)
    assert (c.batch_size, c.block_size, c.precond_rank, c.precond_shift, c.seed) == (100, 100, 100, 1e-6, 0)
    assert (c.sgd_scaling, c.ap_ordering, c.precond_shift_mode) == (W.SGD_UNBIASED, W.AP_GREEDY, W.SHIFT_CALIBRATED)


@pytest.mark.parametrize("n", [0, 1, 511, 512, 513, 100_000, 101_000, 500_000])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_range_partition(W, n, world):
    ranges = [W.shard_range(n, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
        assert a1 == b0
    slot = -(-(-(-n // 512)) // world) * 512 if n else 512  # equal slots of whole chunks
    slot = max(slot, 512)
    for r, (a, b) in enumerate(ranges):
        assert a <= b and (a % 512 == 0 or a == n)  # chunk-aligned: sums independent of world
        assert a == min(r * slot, n) and b - a <= slot  # rank r's slot of the padded buffer
    assert W.shard_padded_rows(n, world) == world * slot >= n


def test_sample_prior_matches_oracle(W, O):
    for kind in (0, 1):
        hw = W.KernelHyperparams(0.7, 1.3, 1e-3, kind)
        ho = O.KernelHyperparams(0.7, 1.3, 1e-3, kind)
        a = W.sample_prior(hw, 5, 300, 42)
        b = O.sample_prior(ho, 5, 300, 42)
        assert np.array_equal(a.frequencies, b.frequencies)
        assert np.array_equal(a.phases, b.phases) and np.array_equal(a.amplitudes, b.amplitudes)
    assert np.array_equal(W.normal_fill(9, 50, 0.1), 0.1 * O.gaussian_vector(9, 50))


def test_cpp_headers_compile_without_gpu():
    """Both C++ test programs (reference-API mirror, Eigen overloads) compile and link here."""
    import subprocess
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2511_16340_b200")
    with tempfile.TemporaryDirectory() as td:
        for src, extra in (("test_gpu_api.cpp", []), ("test_eigen_overloads.cpp",
                                                      ["-I", os.path.join(root, "tests", "cpp", "eigen_shim")])):
            subprocess.run(["g++", "-O1", "-std=c++17", "-I", os.path.join(root, "include"), *extra,
                            os.path.join(root, "tests", "cpp", src), "-L", libdir, "-lwarmgp_b200",
                            f"-Wl,-rpath,{libdir}", "-o", os.path.join(td, src + ".bin")], check=True)


def test_median_heuristic_matches_oracle(W, O):
    """median_heuristic_lengthscale (analysis.cpp:184-203) is host code in the product library:
    same draws and the same order statistic as the oracle, scale-aware (test_analysis.cpp:208-215)."""
    X = O.uniform_inputs(30, 200, 3)
    base = W.median_heuristic_lengthscale(X)
    assert base == O.median_heuristic_lengthscale(X)
    assert 0.1 < base < 2.0
    assert W.median_heuristic_lengthscale(10.0 * X) == pytest.approx(10.0 * base, rel=1e-12)
    X = O.uniform_inputs(31, 1000, 2)
    assert W.median_heuristic_lengthscale(X, 7) == O.median_heuristic_lengthscale(X, 7)

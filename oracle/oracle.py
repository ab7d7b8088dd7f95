"""ctypes binding of the CPU oracle (oracle/libwarmgp_oracle.so).

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg -- never from the product
package ``paper_2511_16340_b200``.  The oracle restates the reference's C++
(/root/reference/proj/core/src/{kernel,solvers,sampling,analysis}.cpp); see
warmgp_oracle.h for the per-function file:line citations.

Arrays follow the reference's Eigen convention: column-major (Fortran order)
float64, right-hand sides as N x s with one RHS per column.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libwarmgp_oracle.so")

MATERN32, RBF = 0, 1
CG, SGD, AP = 0, 1, 2
SGD_UNBIASED, SGD_BLOCK = 0, 1
AP_GREEDY, AP_CYCLIC = 0, 1
SHIFT_CALIBRATED, SHIFT_NOISE_ONLY = 0, 1
OK, INVALID_ARGUMENT, NOT_SPD, DIVERGED = 0, 1, 2, 3


class NotSpdError(RuntimeError):
    """warmgp::NotSpdError (types.hpp:15-18)."""


class DivergenceError(RuntimeError):
    """warmgp::DivergenceError (types.hpp:21-26)."""

    def __init__(self, what: str, iterations: int):
        super().__init__(what)
        self.iterations = iterations


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc only; no reference sources needed)."""
    src = os.path.join(_HERE, "warmgp_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


class Hyp(C.Structure):
    _fields_ = [("kind", C.c_int), ("lengthscale", C.c_double),
                ("signal_scale", C.c_double), ("noise_scale", C.c_double)]


class SolverConfig(C.Structure):
    """warmgp::SolverConfig (solvers.hpp:27-48), reference defaults."""
    _fields_ = [("method", C.c_int), ("tolerance", C.c_double), ("max_iters", C.c_int),
                ("learning_rate", C.c_double), ("momentum", C.c_double),
                ("batch_size", C.c_int64), ("sgd_scaling", C.c_int),
                ("block_size", C.c_int64), ("ap_ordering", C.c_int),
                ("precond_rank", C.c_int64), ("precond_shift", C.c_double),
                ("precond_shift_mode", C.c_int), ("seed", C.c_uint64)]

    def __init__(self, **kw):
        super().__init__()
        lib().wgo_solver_config_default(C.byref(self))
        for k, v in kw.items():
            setattr(self, k, v)


class _Rng(C.Structure):
    _fields_ = [("state", C.c_uint64)]


class _Op(C.Structure):
    pass


_Op._fields_ = [("n", C.c_int64), ("ctx", C.c_void_p), ("matvec", C.c_void_p), ("block", C.c_void_p)]


class _MfCtx(C.Structure):
    _fields_ = [("hyp", Hyp), ("X", C.c_void_p), ("n", C.c_int64), ("d", C.c_int64),
                ("nthreads", C.c_int), ("sq", C.c_void_p)]


class _Precond(C.Structure):
    _fields_ = [("n", C.c_int64), ("k", C.c_int64), ("shift", C.c_double),
                ("L", C.c_void_p), ("cap", C.c_void_p)]


class _Result(C.Structure):
    _fields_ = [("v", C.c_void_p), ("iterations", C.c_int), ("history", C.c_void_p),
                ("history_len", C.c_int), ("converged", C.c_int), ("diverged_at", C.c_int)]


P = C.c_void_p
I64 = C.c_int64
D = C.c_double


def _declare(L):
    sig = {
        "wgo_last_error": (C.c_char_p, []),
        "wgo_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        "wgo_rng_next_u64": (C.c_uint64, [P]),
        "wgo_rng_uniform": (D, [P]),
        "wgo_rng_uniform_range": (D, [P, D, D]),
        "wgo_rng_normal": (D, [P]),
        "wgo_rng_chi_square3": (D, [P]),
        "wgo_rng_uniform_index": (C.c_uint64, [P, C.c_uint64]),
        "wgo_uniform_inputs": (None, [C.c_uint64, I64, I64, P]),
        "wgo_gaussian_vector": (None, [C.c_uint64, I64, P]),
        "wgo_hyp_validate": (C.c_int, [P]),
        "wgo_kernel_from_distance": (D, [P, D]),
        "wgo_pairwise_distances": (C.c_int, [P, I64, P, I64, I64, P]),
        "wgo_gram_matrix": (C.c_int, [P, P, I64, I64, P]),
        "wgo_cross_kernel": (C.c_int, [P, P, I64, P, I64, I64, P]),
        "wgo_extend_assembled": (C.c_int, [P, P, P, I64, P, I64, I64, P]),
        "wgo_kmatvec_rows": (C.c_int, [P, P, I64, I64, P, I64, I64, I64, P, C.c_int]),
        "wgo_cross_matvec": (C.c_int, [P, P, I64, P, I64, I64, P, I64, P, C.c_int]),
        "wgo_solver_config_default": (None, [P]),
        "wgo_op_dense": (None, [P, P, I64]),
        "wgo_op_matrix_free": (C.c_int, [P, P]),
        "wgo_mf_free": (None, [P]),
        "wgo_init_weights": (C.c_int, [C.c_int, P, I64, I64, I64, P]),
        "wgo_relative_residual": (C.c_int, [P, P, P, P]),
        "wgo_quadratic_objective": (D, [P, P, P]),
        "wgo_pivoted_cholesky": (C.c_int, [P, I64, P, P]),
        "wgo_precond_init": (C.c_int, [P, P, I64, I64, D]),
        "wgo_precond_from_op": (C.c_int, [P, P, I64, D, C.c_int]),
        "wgo_precond_apply": (None, [P, P, P]),
        "wgo_precond_free": (None, [P]),
        "wgo_cg_solve_with": (C.c_int, [P, P, C.c_int, P, I64, P, P, P]),
        "wgo_cg_solve": (C.c_int, [P, P, C.c_int, P, I64, P, P]),
        "wgo_sgd_solve": (C.c_int, [P, P, C.c_int, P, I64, P, P]),
        "wgo_ap_solve": (C.c_int, [P, P, C.c_int, P, I64, P, P]),
        "wgo_solve": (C.c_int, [P, P, C.c_int, P, I64, P, P]),
        "wgo_solve_many": (C.c_int, [P, P, I64, C.c_int, P, I64, P, P, P, P, P, P, P, P]),
        "wgo_exact_solve": (C.c_int, [P, I64, P, P]),
        "wgo_rkhs_distance": (D, [P, P, P]),
        "wgo_mll": (C.c_int, [P, P, I64, I64, P, P, P]),
        "wgo_optimize_mll": (C.c_int, [P, P, I64, I64, P, C.c_int, D, P]),
        "wgo_median_heuristic_lengthscale": (D, [P, I64, I64, C.c_uint64]),
        "wgo_sample_prior": (C.c_int, [P, I64, I64, C.c_uint64, P, P, P]),
        "wgo_eval_prior": (C.c_int, [P, P, P, I64, I64, D, P, I64, P]),
        "wgo_build_sample_rhs": (C.c_int, [P, P, P, I64, I64, D, P, I64, D, C.c_uint64, P]),
        "wgo_eval_posterior": (C.c_int, [P, P, P, P, I64, P, I64, I64, P, P, I64, P]),
        "wgo_grad_posterior": (C.c_int, [P, P, P, P, I64, P, I64, I64, P, P, P]),
        "wgo_ascend_peaks": (C.c_int, [P, P, P, P, I64, P, I64, I64, P, P, I64, C.c_int, D, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _check(st: int, iterations: int = 0):
    if st == OK:
        return
    msg = lib().wgo_last_error().decode()
    if st == INVALID_ARGUMENT:
        raise ValueError(msg)
    if st == NOT_SPD:
        raise NotSpdError(msg)
    if st == DIVERGED:
        raise DivergenceError(msg, iterations)
    raise RuntimeError(f"oracle status {st}: {msg}")


# ----------------------------------------------------------------- rng.hpp
def derive_seed(seed: int, stream: int) -> int:
    return int(lib().wgo_derive_seed(seed & (2**64 - 1), stream & (2**64 - 1)))


class Rng:
    """warmgp::Rng (rng.hpp:21-61)."""

    def __init__(self, seed: int):
        self._s = _Rng(seed & (2**64 - 1))

    def next_u64(self) -> int:
        return int(lib().wgo_rng_next_u64(C.byref(self._s)))

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        if lo is None:
            return lib().wgo_rng_uniform(C.byref(self._s))
        return lib().wgo_rng_uniform_range(C.byref(self._s), lo, hi)

    def normal(self) -> float:
        return lib().wgo_rng_normal(C.byref(self._s))

    def chi_square3(self) -> float:
        return lib().wgo_rng_chi_square3(C.byref(self._s))

    def uniform_index(self, n: int) -> int:
        return int(lib().wgo_rng_uniform_index(C.byref(self._s), n))

    def derive(self, stream: int) -> "Rng":
        return Rng(derive_seed(self._s.state, stream))


def uniform_inputs(seed: int, n: int, dim: int) -> np.ndarray:
    X = np.zeros((n, dim), order="F")
    lib().wgo_uniform_inputs(seed & (2**64 - 1), n, dim, _ptr(X))
    return X


def gaussian_vector(seed: int, n: int) -> np.ndarray:
    v = np.zeros(n)
    lib().wgo_gaussian_vector(seed & (2**64 - 1), n, _ptr(v))
    return v


# ----------------------------------------------------------------- kernel
@dataclass
class KernelHyperparams:
    """warmgp::KernelHyperparams (kernel.hpp:8-14); ``kind`` adds the RBF extension."""
    lengthscale: float = 1.0
    signal_scale: float = 1.0
    noise_scale: float = 1e-3
    kind: int = MATERN32

    def c(self) -> Hyp:
        return Hyp(self.kind, self.lengthscale, self.signal_scale, self.noise_scale)


def _hyp(h: KernelHyperparams):
    return C.byref(h.c())


def kernel_from_distance(h: KernelHyperparams, r: float) -> float:
    return lib().wgo_kernel_from_distance(_hyp(h), r)


def kernel(x, xp, h: KernelHyperparams) -> float:
    """matern32(x, x', hyp) (kernel.cpp:23-28), or the RBF map for kind=RBF."""
    x = np.asarray(x, dtype=np.float64)
    xp = np.asarray(xp, dtype=np.float64)
    if x.shape != xp.shape:
        raise ValueError("matern32: dimension mismatch")
    return kernel_from_distance(h, float(np.linalg.norm(x - xp)))


def pairwise_distances(A, B) -> np.ndarray:
    A = _f64(A)
    B = _f64(B)
    D_ = np.zeros((A.shape[0], B.shape[0]), order="F")
    _check(lib().wgo_pairwise_distances(_ptr(A), A.shape[0], _ptr(B), B.shape[0], A.shape[1], _ptr(D_)))
    return D_


def gram_matrix(X, h: KernelHyperparams) -> np.ndarray:
    X = _f64(X)
    n = X.shape[0]
    H = np.zeros((max(n, 0), max(n, 0)), order="F")
    _check(lib().wgo_gram_matrix(_hyp(h), _ptr(X), n, X.shape[1], _ptr(H)))
    return H


def cross_kernel(Xs, X, h: KernelHyperparams) -> np.ndarray:
    Xs = _f64(Xs)
    X = _f64(X)
    if Xs.shape[1] != X.shape[1]:
        raise ValueError("cross_kernel: dimension mismatch")
    K = np.zeros((Xs.shape[0], X.shape[0]), order="F")
    _check(lib().wgo_cross_kernel(_hyp(h), _ptr(Xs), Xs.shape[0], _ptr(X), X.shape[0], X.shape[1], _ptr(K)))
    return K


def extend_assembled(H11, X1, X2, h: KernelHyperparams) -> np.ndarray:
    """extend_system(...).assembled() (kernel.cpp:91-130)."""
    H11 = _f64(H11)
    X1 = _f64(X1)
    X2 = _f64(X2)
    n1, n2 = X1.shape[0], X2.shape[0]
    if n2 > 0 and X2.shape[1] != X1.shape[1]:
        raise ValueError("extend_system: feature dimension mismatch")
    H = np.zeros((n1 + n2, n1 + n2), order="F")
    _check(lib().wgo_extend_assembled(_hyp(h), _ptr(H11), _ptr(X1), n1, _ptr(X2), n2, X1.shape[1], _ptr(H)))
    return H


def kmatvec(X, h: KernelHyperparams, V, rows: tuple[int, int] | None = None, nthreads: int = 0) -> np.ndarray:
    """Matrix-free (K(X,X)+sigma_n^2 I) V over a row range (same entries as gram_matrix)."""
    X = _f64(X)
    V = _f64(V)
    squeeze = V.ndim == 1
    if squeeze:
        V = V.reshape(-1, 1, order="F")
    n = X.shape[0]
    r0, r1 = rows if rows is not None else (0, n)
    Y = np.zeros((r1 - r0, V.shape[1]), order="F")
    _check(lib().wgo_kmatvec_rows(_hyp(h), _ptr(X), n, X.shape[1], _ptr(V), V.shape[1], r0, r1, _ptr(Y), nthreads))
    return Y[:, 0] if squeeze else Y


def cross_matvec(Xs, X, h: KernelHyperparams, W, nthreads: int = 0) -> np.ndarray:
    Xs = _f64(Xs)
    X = _f64(X)
    W = _f64(W)
    squeeze = W.ndim == 1
    if squeeze:
        W = W.reshape(-1, 1, order="F")
    Y = np.zeros((Xs.shape[0], W.shape[1]), order="F")
    _check(lib().wgo_cross_matvec(_hyp(h), _ptr(Xs), Xs.shape[0], _ptr(X), X.shape[0], X.shape[1],
                                  _ptr(W), W.shape[1], _ptr(Y), nthreads))
    return Y[:, 0] if squeeze else Y


# ----------------------------------------------------------------- operators
class Operator:
    """Dense H (the reference's representation) or the matrix-free kernel operator."""

    def __init__(self, H=None, X=None, hyp: KernelHyperparams | None = None, nthreads: int = 0):
        self._op = _Op()
        self._keep = []
        if H is not None:
            H = _f64(H)
            self._keep.append(H)
            lib().wgo_op_dense(C.byref(self._op), _ptr(H), H.shape[0])
            self.n = H.shape[0]
            self._mf = None
        else:
            X = _f64(X)
            self._keep.append(X)
            self._mf = _MfCtx(hyp.c(), X.ctypes.data, X.shape[0], X.shape[1], nthreads, None)
            _check(lib().wgo_op_matrix_free(C.byref(self._op), C.byref(self._mf)))
            self.n = X.shape[0]

    @property
    def ref(self):
        return C.byref(self._op)

    def __del__(self):
        try:
            if self._mf is not None and self._mf.sq:
                lib().wgo_mf_free(C.byref(self._mf))
        except Exception:
            pass


def _as_op(H) -> Operator:
    return H if isinstance(H, Operator) else Operator(H=H)


# ----------------------------------------------------------------- solvers
@dataclass
class Initialization:
    """warmgp::Initialization (solvers.hpp:52-63)."""
    warm_start: bool = False
    u1: np.ndarray | None = None

    @staticmethod
    def cold() -> "Initialization":
        return Initialization()

    @staticmethod
    def warm(u1) -> "Initialization":
        return Initialization(True, np.asarray(u1, dtype=np.float64).copy())


@dataclass
class SolveResult:
    """warmgp::SolveResult (solvers.hpp:102-109)."""
    v: np.ndarray
    iterations: int
    residual_history: list
    converged: bool

    def final_residual(self) -> float:
        return self.residual_history[-1]


def init_weights(init: Initialization, n1: int, n2: int) -> np.ndarray:
    v = np.zeros(max(n1 + n2, 0))
    u1 = None if init.u1 is None else np.ascontiguousarray(init.u1, dtype=np.float64)
    _check(lib().wgo_init_weights(int(init.warm_start), _ptr(u1), 0 if u1 is None else u1.size, n1, n2, _ptr(v)))
    return v


def relative_residual(H, v, b) -> float:
    op = _as_op(H)
    v = _f64(v)
    b = _f64(b)
    out = C.c_double()
    _check(lib().wgo_relative_residual(op.ref, _ptr(v), _ptr(b), C.byref(out)))
    return out.value


def quadratic_objective(H, v, b) -> float:
    op = _as_op(H)
    return lib().wgo_quadratic_objective(op.ref, _ptr(_f64(v)), _ptr(_f64(b)))


def pivoted_cholesky(H, rank: int) -> np.ndarray:
    op = _as_op(H)
    L = np.zeros((op.n, max(rank, 0)), order="F")
    ach = C.c_int64()
    _check(lib().wgo_pivoted_cholesky(op.ref, rank, _ptr(L), C.byref(ach)))
    return np.asfortranarray(L[:, : ach.value])


class CgPreconditioner:
    """warmgp::CgPreconditioner (solvers.hpp:82-100)."""

    def __init__(self, L=None, shift: float = 1.0, _raw: _Precond | None = None):
        if _raw is not None:
            self._p = _raw
            return
        self._p = _Precond()
        L = _f64(L)
        _check(lib().wgo_precond_init(C.byref(self._p), _ptr(L), L.shape[0], L.shape[1], shift))

    @staticmethod
    def from_matrix(H, rank: int, shift: float, mode: int = SHIFT_CALIBRATED) -> "CgPreconditioner":
        op = _as_op(H)
        p = _Precond()
        _check(lib().wgo_precond_from_op(C.byref(p), op.ref, rank, shift, mode))
        return CgPreconditioner(_raw=p)

    @property
    def rank(self) -> int:
        return self._p.k

    @property
    def shift(self) -> float:
        return self._p.shift

    def apply(self, r) -> np.ndarray:
        r = _f64(r)
        z = np.zeros_like(r)
        lib().wgo_precond_apply(C.byref(self._p), _ptr(r), _ptr(z))
        return z

    def __del__(self):
        try:
            lib().wgo_precond_free(C.byref(self._p))
        except Exception:
            pass


def _run_single(fn, H, b, init: Initialization, cfg: SolverConfig, *extra) -> SolveResult:
    op = _as_op(H)
    b = _f64(b)
    n = op.n
    v = np.zeros(n)
    hist = np.zeros(cfg.max_iters + 1)
    res = _Result(v.ctypes.data, 0, hist.ctypes.data, 0, 0, 0)
    u1 = None if not init.warm_start else np.ascontiguousarray(init.u1, dtype=np.float64)
    n1 = 0 if u1 is None else u1.size
    st = fn(op.ref, _ptr(b), int(init.warm_start), _ptr(u1), n1, C.byref(cfg), *extra, C.byref(res))
    _check(st, res.diverged_at)
    return SolveResult(v, res.iterations, hist[: res.history_len].tolist(), bool(res.converged))


def cg_solve_with(H, b, init, cfg, precond: CgPreconditioner) -> SolveResult:
    return _run_single(lib().wgo_cg_solve_with, H, b, init, cfg, C.byref(precond._p))


def cg_solve(H, b, init, cfg) -> SolveResult:
    return _run_single(lib().wgo_cg_solve, H, b, init, cfg)


def sgd_solve(H, b, init, cfg) -> SolveResult:
    return _run_single(lib().wgo_sgd_solve, H, b, init, cfg)


def ap_solve(H, b, init, cfg) -> SolveResult:
    return _run_single(lib().wgo_ap_solve, H, b, init, cfg)


def solve(H, b, init, cfg) -> SolveResult:
    return _run_single(lib().wgo_solve, H, b, init, cfg)


def solve_many(H, rhs, inits: list, cfg: SolverConfig) -> list:
    """solve_many (solvers.cpp:321-354).  Raises like the reference at the first failing column."""
    op = _as_op(H)
    B = _f64(rhs)
    if B.ndim == 1:
        B = B.reshape(-1, 1, order="F")
    s = B.shape[1]
    if len(inits) != s:
        raise ValueError("solve_many: one initialization per right-hand side required")
    warm = all(i.warm_start for i in inits) if s else False
    if any(i.warm_start for i in inits) and not warm:
        # Mixed warm/cold: run column by column (the C oracle takes one mode per call).
        return [_solve_col(op, B[:, i], inits[i], cfg, i) for i in range(s)]
    n = op.n
    n1 = inits[0].u1.size if warm else 0
    U1 = np.asfortranarray(np.stack([i.u1 for i in inits], axis=1)) if warm else None
    V = np.zeros((n, s), order="F")
    hs = cfg.max_iters + 1
    hist = np.zeros((s, hs))
    its = np.zeros(s, dtype=np.int32)
    hl = np.zeros(s, dtype=np.int32)
    cv = np.zeros(s, dtype=np.int32)
    dv = np.zeros(s, dtype=np.int32)
    fc = C.c_int(-1)
    st = lib().wgo_solve_many(op.ref, _ptr(B), s, int(warm), _ptr(U1), n1, C.byref(cfg), _ptr(V),
                              _ptr(its), _ptr(hist), _ptr(hl), _ptr(cv), C.byref(fc), _ptr(dv))
    if st:
        _check(st, int(dv[fc.value]) if fc.value >= 0 else 0)
    return [SolveResult(V[:, i].copy(), int(its[i]), hist[i, : hl[i]].tolist(), bool(cv[i])) for i in range(s)]


def _solve_col(op, b, init, cfg, i):
    c = SolverConfig()
    C.memmove(C.byref(c), C.byref(cfg), C.sizeof(SolverConfig))
    if cfg.method == SGD:
        c.seed = derive_seed(cfg.seed, i)
    if cfg.method == CG:
        pre = CgPreconditioner.from_matrix(op, cfg.precond_rank, cfg.precond_shift, cfg.precond_shift_mode)
        return cg_solve_with(op, b, init, c, pre)
    return solve(op, b, init, c)


def exact_solve(H, b) -> np.ndarray:
    H = _f64(H)
    b = _f64(b)
    x = np.zeros_like(b)
    _check(lib().wgo_exact_solve(_ptr(H), H.shape[0], _ptr(b), _ptr(x)))
    return x


def rkhs_distance(H, v_init, v_exact) -> float:
    op = _as_op(H)
    return lib().wgo_rkhs_distance(op.ref, _ptr(_f64(v_init)), _ptr(_f64(v_exact)))


@dataclass
class MllResult:
    """warmgp::MllResult (analysis.hpp:42-45)."""
    value: float
    grad: np.ndarray  # d/d(log l, log s_f, log sigma_n)


def mll(X, y, h: KernelHyperparams) -> MllResult:
    """mll (analysis.cpp:99-139)."""
    X = _f64(X)
    y = _f64(y).ravel()
    if X.shape[0] != y.shape[0]:
        raise ValueError("mll: X rows != y length")
    val = C.c_double(0.0)
    g = np.zeros(3)
    _check(lib().wgo_mll(_hyp(h), _ptr(X), X.shape[0], X.shape[1], _ptr(y), C.byref(val), _ptr(g)))
    return MllResult(val.value, g)


def optimize_mll(X, y, init: KernelHyperparams, steps: int, step_size: float) -> KernelHyperparams:
    """optimize_mll (analysis.cpp:141-182)."""
    X = _f64(X)
    y = _f64(y).ravel()
    out = Hyp()
    _check(lib().wgo_optimize_mll(_hyp(init), _ptr(X), X.shape[0], X.shape[1], _ptr(y), steps,
                                  step_size, C.byref(out)))
    return KernelHyperparams(out.lengthscale, out.signal_scale, out.noise_scale, out.kind)


def median_heuristic_lengthscale(X, seed: int = 0) -> float:
    """median_heuristic_lengthscale (analysis.cpp:184-203)."""
    X = _f64(X)
    return lib().wgo_median_heuristic_lengthscale(_ptr(X), X.shape[0], X.shape[1], seed & (2**64 - 1))


# ----------------------------------------------------------------- sampling
@dataclass
class RffPrior:
    """warmgp::RffPrior (sampling.hpp:14-22)."""
    frequencies: np.ndarray  # F x D
    phases: np.ndarray
    amplitudes: np.ndarray
    signal_scale: float = 1.0

    @property
    def num_features(self) -> int:
        return self.frequencies.shape[0]

    @property
    def dim(self) -> int:
        return self.frequencies.shape[1]


def sample_prior(h: KernelHyperparams, dim: int, num_features: int, seed: int) -> RffPrior:
    if dim < 1 or num_features < 1:
        raise ValueError("sample_prior: dim and num_features must be positive")
    Om = np.zeros((num_features, dim), order="F")
    ph = np.zeros(num_features)
    am = np.zeros(num_features)
    _check(lib().wgo_sample_prior(_hyp(h), dim, num_features, seed & (2**64 - 1), _ptr(Om), _ptr(ph), _ptr(am)))
    return RffPrior(Om, ph, am, h.signal_scale)


def eval_prior(p: RffPrior, Xs) -> np.ndarray:
    Xs = _f64(Xs)
    if Xs.shape[1] != p.dim:
        raise ValueError("eval_prior: dimension mismatch")
    Om = _f64(p.frequencies)
    out = np.zeros(Xs.shape[0])
    _check(lib().wgo_eval_prior(_ptr(Om), _ptr(_f64(p.phases)), _ptr(_f64(p.amplitudes)), p.num_features,
                                p.dim, p.signal_scale, _ptr(Xs), Xs.shape[0], _ptr(out)))
    return out


def build_sample_rhs(p: RffPrior, X, noise_scale: float, seed: int) -> np.ndarray:
    X = _f64(X)
    Om = _f64(p.frequencies)
    out = np.zeros(X.shape[0])
    _check(lib().wgo_build_sample_rhs(_ptr(Om), _ptr(_f64(p.phases)), _ptr(_f64(p.amplitudes)), p.num_features,
                                      p.dim, p.signal_scale, _ptr(X), X.shape[0], noise_scale,
                                      seed & (2**64 - 1), _ptr(out)))
    return out


def eval_posterior(h: KernelHyperparams, p: RffPrior, X_train, weights, Xs) -> np.ndarray:
    X_train = _f64(X_train)
    weights = _f64(weights)
    Xs = _f64(Xs)
    if weights.size != X_train.shape[0]:
        raise ValueError("eval_posterior: weights length != training rows")
    Om = _f64(p.frequencies)
    out = np.zeros(Xs.shape[0])
    _check(lib().wgo_eval_posterior(_hyp(h), _ptr(Om), _ptr(_f64(p.phases)), _ptr(_f64(p.amplitudes)),
                                    p.num_features, _ptr(X_train), X_train.shape[0], X_train.shape[1],
                                    _ptr(weights), _ptr(Xs), Xs.shape[0], _ptr(out)))
    return out


def grad_posterior(h: KernelHyperparams, p: RffPrior, X_train, weights, x) -> np.ndarray:
    """grad_posterior (sampling.cpp:77-87) at one point."""
    X_train = _f64(X_train)
    x = np.ascontiguousarray(x, dtype=np.float64)
    g = np.zeros(x.size)
    _check(lib().wgo_grad_posterior(_hyp(h), _ptr(_f64(p.frequencies)), _ptr(_f64(p.phases)),
                                    _ptr(_f64(p.amplitudes)), p.num_features, _ptr(X_train),
                                    X_train.shape[0], x.size, _ptr(_f64(weights)), _ptr(x), _ptr(g)))
    return g


def ascend_peaks(h: KernelHyperparams, p: RffPrior, X_train, weights, starts, steps: int, rate: float):
    """ascend_peaks (thompson.cpp:209-258) for one posterior sample -> (best point, value)."""
    X_train = _f64(X_train)
    starts = _f64(starts)
    dim = starts.shape[1]
    bx = np.zeros(dim)
    bv = C.c_double(0.0)
    _check(lib().wgo_ascend_peaks(_hyp(h), _ptr(_f64(p.frequencies)), _ptr(_f64(p.phases)),
                                  _ptr(_f64(p.amplitudes)), p.num_features, _ptr(X_train),
                                  X_train.shape[0], dim, _ptr(_f64(weights)), _ptr(starts),
                                  starts.shape[0], steps, rate, _ptr(bx), C.byref(bv)))
    return bx, bv.value

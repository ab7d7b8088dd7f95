"""Python mirror of the reference's warmgp API over the C-ABI of libwarmgp_b200.so.

The reference (/root/reference/proj) is a C++ library whose boundary is the
free-function API of warmgp::{kernel,solvers,sampling}.hpp; its C++ mirror over
this ABI is include/warmgp/gpu.hpp.  This module offers the same names to Python
callers (tests, bench.py) -- a thin ctypes layer, no compute of its own:

    reference (dense H)                           here (matrix-free device operator)
    gram_matrix(X, hyp)          kernel.cpp:48    KernelOperator(hyp, X)
    extend_system(prev, X2, ..)  kernel.cpp:108   op.append_rows(X2)
    H * V                        solvers.cpp:162  op.kmatvec(V)
    solve_many(H, rhs, inits, cfg) solvers.cpp:321 solve_many(op, rhs, inits, cfg)
    cg_solve / sgd_solve / ap_solve / solve       same names
    pivoted_cholesky(H, rank)    solvers.cpp:72   pivoted_cholesky(op, rank)

Errors map like the reference's exceptions (types.hpp:15-32): NotSpdError,
DivergenceError(iterations), ValueError for std::invalid_argument.  There is no
CPU fallback: a missing library or GPU raises ExtensionUnavailable.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# WGP_LIB_PATH: an alternative build of the same library (A/B probes only)
LIB_PATH = os.environ.get("WGP_LIB_PATH") or os.path.join(_HERE, "libwarmgp_b200.so")

MATERN32, RBF = 0, 1
F64, F32_3XTF32, TF32, F32_SIMT = 0, 1, 2, 3
CG, SGD, AP = 0, 1, 2
SGD_UNBIASED, SGD_BLOCK = 0, 1
AP_GREEDY, AP_CYCLIC = 0, 1
SHIFT_CALIBRATED, SHIFT_NOISE_ONLY = 0, 1
RESIDUAL_DIRECT, RESIDUAL_ANCHORED = 0, 1
OK, INVALID_ARGUMENT, NOT_SPD, DIVERGED, CUDA_ERROR, NCCL_ERROR, OOM = range(7)

# Every symbol include/warmgp_capi.h declares (checked by tests/test_capi_abi.py).
EXPORTS = (
    "wgp_abi_version", "wgp_last_error", "wgp_solver_config_default", "wgp_shard_range",
    "wgp_ctx_create", "wgp_nccl_unique_id", "wgp_ctx_create_sharded", "wgp_ctx_destroy",
    "wgp_allgather_rows_dev",
    "wgp_ctx_stream", "wgp_op_create", "wgp_op_destroy", "wgp_op_append_rows", "wgp_op_size",
    "wgp_op_dim", "wgp_op_precision", "wgp_kmatvec", "wgp_kmatvec_dev", "wgp_kmatvec_sharded_dev",
    "wgp_residual_dev",
    "wgp_cross_matvec", "wgp_solve_many", "wgp_solve", "wgp_pivoted_cholesky", "wgp_precond_info",
    "wgp_rff_eval", "wgp_derive_seed", "wgp_rng_next_u64", "wgp_rng_uniform", "wgp_rng_normal",
    "wgp_rng_chi_square3", "wgp_rng_uniform_index", "wgp_normal_fill", "wgp_sample_prior",
    "wgp_rng_normal_fill", "wgp_kernel_timer_enable", "wgp_kernel_timer_read", "wgp_rff_eval_fast",
    "wgp_exact_solve", "wgp_grad_posterior", "wgp_ascend_peaks",
    "wgp_mll", "wgp_optimize_mll", "wgp_median_heuristic_lengthscale",
    "wgp_axpy_cols_dev", "wgp_xpby_cols_dev", "wgp_coldots_dev",
    "wgp_op_set_residual_mode", "wgp_op_residual_mode", "wgp_op_last_anchor_count",
    "wgp_loopback_group_create", "wgp_loopback_group_destroy", "wgp_ctx_create_loopback",
    "wgp_shard_padded_rows",
    "wgp_precond_create", "wgp_precond_create_from_factor", "wgp_precond_destroy", "wgp_precond_get",
    "wgp_precond_apply", "wgp_cg_solve_with", "wgp_cross_kernel", "wgp_relative_residual",
    "wgp_quadratic_objective", "wgp_init_weights", "wgp_build_sample_rhs", "wgp_kernel_timer_read_tag",
    "wgp_posterior_select",
)


class ExtensionUnavailable(RuntimeError):
    """The CUDA library is missing or cannot run (no silent fallback exists)."""


class NotSpdError(RuntimeError):
    """warmgp::NotSpdError (types.hpp:15-18)."""


class DivergenceError(RuntimeError):
    """warmgp::DivergenceError (types.hpp:21-26)."""

    def __init__(self, what: str, iterations: int):
        super().__init__(what)
        self.iterations = iterations


class CudaError(RuntimeError):
    pass


class SolverConfig(C.Structure):
    """warmgp::SolverConfig (solvers.hpp:27-48), defaults from wgp_solver_config_default."""
    _fields_ = [("method", C.c_int32), ("tolerance", C.c_double), ("max_iters", C.c_int32),
                ("learning_rate", C.c_double), ("momentum", C.c_double),
                ("batch_size", C.c_int64), ("sgd_scaling", C.c_int32),
                ("block_size", C.c_int64), ("ap_ordering", C.c_int32),
                ("precond_rank", C.c_int64), ("precond_shift", C.c_double),
                ("precond_shift_mode", C.c_int32), ("seed", C.c_uint64)]

    def __init__(self, **kw):
        super().__init__()
        lib().wgp_solver_config_default(C.byref(self))
        for k, v in kw.items():
            setattr(self, k, v)

    def copy(self, **kw) -> "SolverConfig":
        c = SolverConfig()
        C.memmove(C.byref(c), C.byref(self), C.sizeof(SolverConfig))
        for k, v in kw.items():
            setattr(c, k, v)
        return c


P = C.c_void_p
I64 = C.c_int64
D = C.c_double
_lib = None


def _declare(L):
    sig = {
        "wgp_abi_version": (C.c_int, []),
        "wgp_last_error": (C.c_char_p, []),
        "wgp_solver_config_default": (None, [P]),
        "wgp_shard_range": (None, [I64, C.c_int, C.c_int, P, P]),
        "wgp_ctx_create": (C.c_int, [C.c_int, P]),
        "wgp_nccl_unique_id": (C.c_int, [P]),
        "wgp_ctx_create_sharded": (C.c_int, [C.c_int, C.c_int, C.c_int, P, P]),
        "wgp_loopback_group_create": (C.c_int, [C.c_int, P]),
        "wgp_loopback_group_destroy": (None, [P]),
        "wgp_ctx_create_loopback": (C.c_int, [C.c_int, C.c_int, P, P]),
        "wgp_shard_padded_rows": (I64, [I64, C.c_int]),
        "wgp_precond_create": (C.c_int, [P, I64, D, C.c_int, P]),
        "wgp_precond_create_from_factor": (C.c_int, [P, P, I64, I64, D, P]),
        "wgp_precond_destroy": (None, [P]),
        "wgp_precond_get": (C.c_int, [P, P, P]),
        "wgp_precond_apply": (C.c_int, [P, P, I64, C.c_int, P, I64]),
        "wgp_cg_solve_with": (C.c_int, [P, P, P, P, I64, C.c_int, P, I64, I64, P, I64, P, P, I64, P, P]),
        "wgp_cross_kernel": (C.c_int, [P, P, I64, I64, P, I64]),
        "wgp_relative_residual": (C.c_int, [P, P, I64, P, I64, C.c_int, P]),
        "wgp_quadratic_objective": (C.c_int, [P, P, I64, P, I64, C.c_int, P]),
        "wgp_init_weights": (C.c_int, [P, I64, I64, P]),
        "wgp_build_sample_rhs": (C.c_int, [P, P, P, P, C.c_int, D, D, C.c_uint64, P]),
        "wgp_ctx_destroy": (None, [P]),
        "wgp_allgather_rows_dev": (C.c_int, [P, P, I64, C.c_int, P]),
        "wgp_ctx_stream": (P, [P]),
        "wgp_op_create": (C.c_int, [P, C.c_int, D, D, D, C.c_int, C.c_int, P]),
        "wgp_op_destroy": (None, [P]),
        "wgp_op_append_rows": (C.c_int, [P, P, I64, I64, C.c_int]),
        "wgp_op_size": (I64, [P]),
        "wgp_op_dim": (C.c_int, [P]),
        "wgp_op_precision": (C.c_int, [P]),
        "wgp_op_set_residual_mode": (C.c_int, [P, C.c_int]),
        "wgp_op_residual_mode": (C.c_int, [P]),
        "wgp_op_last_anchor_count": (C.c_int, [P]),
        "wgp_kmatvec": (C.c_int, [P, P, I64, C.c_int, P, I64]),
        "wgp_kmatvec_dev": (C.c_int, [P, P, P, C.c_int, P]),
        "wgp_kmatvec_sharded_dev": (C.c_int, [P, P, P, C.c_int, P]),
        "wgp_residual_dev": (C.c_int, [P, P, P, P, C.c_int, P]),
        "wgp_axpy_cols_dev": (C.c_int, [P, P, P, P, I64, C.c_int, P]),
        "wgp_xpby_cols_dev": (C.c_int, [P, P, P, P, P, I64, C.c_int, P]),
        "wgp_coldots_dev": (C.c_int, [P, P, P, I64, C.c_int, P, P, P]),
        "wgp_cross_matvec": (C.c_int, [P, P, I64, I64, P, I64, C.c_int, P, I64]),
        "wgp_solve_many": (C.c_int, [P, P, P, I64, C.c_int, P, I64, I64, P, I64, P, P, I64, P, P,
                                     P, P]),
        "wgp_solve": (C.c_int, [P, P, P, P, I64, P, P, P, P, P, P]),
        "wgp_pivoted_cholesky": (C.c_int, [P, I64, P, I64, P]),
        "wgp_precond_info": (C.c_int, [P, I64, D, C.c_int, P, P]),
        "wgp_rff_eval": (C.c_int, [P, P, P, P, C.c_int, C.c_int, D, P, I64, I64, P, I64]),
        "wgp_rff_eval_fast": (C.c_int, [P, P, P, P, C.c_int, C.c_int, D, P, I64, I64, P, I64]),
        "wgp_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        "wgp_rng_next_u64": (C.c_uint64, [P]),
        "wgp_rng_uniform": (D, [P]),
        "wgp_rng_normal": (D, [P]),
        "wgp_rng_chi_square3": (D, [P]),
        "wgp_rng_uniform_index": (C.c_uint64, [P, C.c_uint64]),
        "wgp_normal_fill": (None, [C.c_uint64, I64, D, P]),
        "wgp_rng_normal_fill": (None, [P, I64, D, P]),
        "wgp_kernel_timer_enable": (None, [C.c_int]),
        "wgp_exact_solve": (C.c_int, [P, P, I64, C.c_int, P, I64]),
        "wgp_mll": (C.c_int, [P, P, P, P, P]),
        "wgp_optimize_mll": (C.c_int, [P, P, P, C.c_int, D, P]),
        "wgp_median_heuristic_lengthscale": (D, [P, I64, I64, C.c_int, C.c_uint64]),
        "wgp_grad_posterior": (C.c_int, [P, P, P, P, C.c_int, C.c_int, D, P, I64, P, I64, P, I64, P, I64]),
        "wgp_ascend_peaks": (C.c_int, [P, P, P, P, C.c_int, C.c_int, D, P, I64, P, C.c_int, C.c_int, D, P, P]),
        "wgp_kernel_timer_read": (C.c_int, [P, P]),
        "wgp_kernel_timer_read_tag": (C.c_int, [C.c_char_p, P, P]),
        "wgp_posterior_select": (C.c_int, [P, P, P, P, C.c_int, C.c_int, D, P, I64, P, I64, I64, C.c_int,
                                          C.c_int, P]),
        "wgp_sample_prior": (C.c_int, [C.c_int, D, I64, I64, C.c_uint64, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def lib():
    """Load libwarmgp_b200.so (fails loudly when it is missing: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionUnavailable(
                f"{LIB_PATH} is missing; build it with `python -m paper_2511_16340_b200.build`")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def _check(st: int, iterations: int = 0):
    if st == OK:
        return
    msg = lib().wgp_last_error().decode(errors="replace")
    if st == INVALID_ARGUMENT:
        raise ValueError(msg)
    if st == NOT_SPD:
        raise NotSpdError(msg)
    if st == DIVERGED:
        raise DivergenceError(msg, iterations)
    if st == OOM:
        raise MemoryError(msg)
    if st == CUDA_ERROR:
        raise CudaError(msg)
    raise RuntimeError(f"wgp status {st}: {msg}")


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    a, b = C.c_int64(), C.c_int64()
    lib().wgp_shard_range(n, world, rank, C.byref(a), C.byref(b))
    return a.value, b.value


def shard_padded_rows(n: int, world: int) -> int:
    """Rows of a full buffer exchanged by allgather_rows_dev (world equal slots)."""
    return int(lib().wgp_shard_padded_rows(n, world))


@dataclass
class KernelHyperparams:
    """warmgp::KernelHyperparams (kernel.hpp:8-14) + ``kind`` (RBF extension)."""
    lengthscale: float = 1.0
    signal_scale: float = 1.0
    noise_scale: float = 1e-3
    kind: int = MATERN32


class LoopbackGroup:
    """`world` ranks emulated by threads of this process on one device
    (wgp_loopback_group_create): each thread creates DeviceContext(device, rank,
    loopback=group) and runs the sharded calls; collectives are host barriers plus
    device-to-device copies (correctness testing of the sharded path, not a performance
    configuration).  The library calls release the GIL, so the rank threads run
    concurrently."""

    def __init__(self, world: int):
        self._h = C.c_void_p()
        _check(lib().wgp_loopback_group_create(int(world), C.byref(self._h)))
        self.world = int(world)

    def __del__(self):
        try:
            if self._h:
                lib().wgp_loopback_group_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


class DeviceContext:
    """One CUDA device (one process per GPU); optionally a NCCL row-sharded group."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, unique_id: bytes | None = None,
                 loopback: "LoopbackGroup | None" = None):
        self._h = C.c_void_p()
        self._group = loopback  # keeps the group alive while this context exists
        if loopback is not None:
            world = loopback.world
            _check(lib().wgp_ctx_create_loopback(device, rank, loopback._h, C.byref(self._h)))
        elif world == 1:
            _check(lib().wgp_ctx_create(device, C.byref(self._h)))
        else:
            buf = C.create_string_buffer(bytes(unique_id), 128)
            _check(lib().wgp_ctx_create_sharded(device, rank, world, buf, C.byref(self._h)))
        self.device, self.rank, self.world = device, rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().wgp_nccl_unique_id(buf))
        return buf.raw

    def allgather_rows_dev(self, dV_ptr: int, n: int, s: int, stream: int = 0):
        """In-place all-gather of this group's row slices of a full fp64 buffer with
        shard_padded_rows(n, world) x s rows."""
        _check(lib().wgp_allgather_rows_dev(self._h, C.c_void_p(dV_ptr), n, s,
                                            C.c_void_p(stream) if stream else None))

    # fused solver vector kernels on device [n][s] row-major fp64 buffers (solvers.cpp:163-180)
    def axpy_cols_dev(self, dY: int, dX: int, dAlpha: int, n: int, s: int, stream: int = 0):
        _check(lib().wgp_axpy_cols_dev(self._h, C.c_void_p(dY), C.c_void_p(dX), C.c_void_p(dAlpha),
                                       n, s, C.c_void_p(stream)))

    def xpby_cols_dev(self, dP: int, dZ: int, dBeta: int, dActive: int, n: int, s: int, stream: int = 0):
        _check(lib().wgp_xpby_cols_dev(self._h, C.c_void_p(dP), C.c_void_p(dZ), C.c_void_p(dBeta),
                                       C.c_void_p(dActive), n, s, C.c_void_p(stream)))

    def coldots_dev(self, dA: int, dB: int, n: int, s: int, dOut: int, dWork: int, stream: int = 0):
        """dWork: at least ceil(n / 512) * s fp64."""
        _check(lib().wgp_coldots_dev(self._h, C.c_void_p(dA), C.c_void_p(dB), n, s, C.c_void_p(dOut),
                                     C.c_void_p(dWork), C.c_void_p(stream)))

    @property
    def stream(self) -> int:
        return lib().wgp_ctx_stream(self._h) or 0

    def close(self):
        if self._h:
            lib().wgp_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: DeviceContext | None = None


def default_context() -> DeviceContext:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = DeviceContext(0)
    return _default_ctx


class KernelOperator:
    """Matrix-free H = K(X, X) + sigma_n^2 I resident on the device.

    Replaces CovarianceMatrix / gram_matrix (kernel.hpp:25-38): X lives on the
    GPU, H is never materialised.  ``append_rows`` is extend_system's growth step.
    """

    def __init__(self, hyp: KernelHyperparams, X=None, dim: int | None = None,
                 precision: int = F64, ctx: DeviceContext | None = None,
                 residual: int = RESIDUAL_DIRECT):
        self.ctx = ctx or default_context()
        self.hyp = hyp
        if X is not None:
            X = _f64(X)
            if X.ndim != 2:
                raise ValueError("X must be 2-d (n x dim)")
            dim = X.shape[1]
        self._h = C.c_void_p()
        _check(lib().wgp_op_create(self.ctx._h, hyp.kind, hyp.lengthscale, hyp.signal_scale,
                                   hyp.noise_scale, precision, int(dim), C.byref(self._h)))
        self.dim = int(dim)
        self.precision = precision
        if residual != RESIDUAL_DIRECT:
            self.residual_mode = residual
        if X is not None and X.shape[0] > 0:
            self.append_rows(X)

    def append_rows(self, X2):
        X2 = _f64(X2)
        if X2.ndim != 2 or (X2.shape[0] > 0 and X2.shape[1] != self.dim):
            raise ValueError("extend_system: feature dimension mismatch")
        _check(lib().wgp_op_append_rows(self._h, _ptr(X2), X2.shape[0], max(X2.shape[0], 1), 1))

    @property
    def n(self) -> int:
        return int(lib().wgp_op_size(self._h))

    @property
    def residual_mode(self) -> int:
        """CG true-residual mode (RESIDUAL_DIRECT / RESIDUAL_ANCHORED, warmgp_capi.h)."""
        return int(lib().wgp_op_residual_mode(self._h))

    @residual_mode.setter
    def residual_mode(self, mode: int):
        _check(lib().wgp_op_set_residual_mode(self._h, int(mode)))

    @property
    def last_anchor_count(self) -> int:
        """fp64 anchor evaluations made by the last CG solve (RESIDUAL_ANCHORED)."""
        return int(lib().wgp_op_last_anchor_count(self._h))

    def size(self) -> int:
        return self.n

    def kmatvec(self, V, out=None) -> np.ndarray:
        """(K(X,X) + sigma_n^2 I) V for host V (n or n x s); ``out``: optional
        Fortran-ordered n x s float64 destination (e.g. a pinned buffer)."""
        V = _f64(V)
        squeeze = V.ndim == 1
        if squeeze:
            V = V.reshape(-1, 1, order="F")
        n = self.n
        if V.shape[0] != n:
            raise ValueError("kmatvec: V rows != operator size")
        if out is None:
            Y = np.zeros((n, V.shape[1]), order="F")
        else:
            Y = out
            if Y.shape != V.shape or Y.dtype != np.float64 or not Y.flags.f_contiguous:
                raise ValueError("kmatvec: out must be a Fortran-ordered float64 n x s array")
        _check(lib().wgp_kmatvec(self._h, _ptr(V), n, V.shape[1], _ptr(Y), n))
        return Y[:, 0] if squeeze else Y

    def kmatvec_dev(self, dV_ptr: int, dY_ptr: int, s: int, stream: int = 0):
        _check(lib().wgp_kmatvec_dev(self._h, C.c_void_p(dV_ptr), C.c_void_p(dY_ptr), s,
                                     C.c_void_p(stream) if stream else None))

    def kmatvec_sharded_dev(self, dV_ptr: int, dY_ptr: int, s: int, stream: int = 0):
        """Row-sharded H V: dV the padded full-row buffer with this rank's slot current; the
        slots are all-gathered while the local diagonal block computes; dY this rank's rows."""
        _check(lib().wgp_kmatvec_sharded_dev(self._h, C.c_void_p(dV_ptr), C.c_void_p(dY_ptr), s,
                                             C.c_void_p(stream) if stream else None))

    def residual_dev(self, dB_ptr: int, dV_ptr: int, dY_ptr: int, s: int, stream: int = 0):
        _check(lib().wgp_residual_dev(self._h, C.c_void_p(dB_ptr), C.c_void_p(dV_ptr),
                                      C.c_void_p(dY_ptr), s, C.c_void_p(stream) if stream else None))

    def cross_matvec(self, Xs, W) -> np.ndarray:
        """K(X*, X) W without the noise term (cross_kernel kernel.cpp:74-89 times weights)."""
        Xs = _f64(Xs)
        W = _f64(W)
        squeeze = W.ndim == 1
        if squeeze:
            W = W.reshape(-1, 1, order="F")
        if Xs.shape[1] != self.dim:
            raise ValueError("cross_kernel: dimension mismatch")
        m = Xs.shape[0]
        Y = np.zeros((m, W.shape[1]), order="F")
        _check(lib().wgp_cross_matvec(self._h, _ptr(Xs), m, max(m, 1), _ptr(W), self.n, W.shape[1],
                                      _ptr(Y), max(m, 1)))
        return Y[:, 0] if squeeze else Y

    def close(self):
        if self._h:
            lib().wgp_op_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gram_operator(X, hyp: KernelHyperparams, precision: int = F64, ctx=None) -> KernelOperator:
    """Device counterpart of gram_matrix (kernel.cpp:48-72)."""
    X = _f64(X)
    if X.shape[0] < 1:
        raise ValueError("gram_matrix: need at least one row")
    return KernelOperator(hyp, X, precision=precision, ctx=ctx)


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
    residual_history: list = field(default_factory=list)
    converged: bool = False

    def final_residual(self) -> float:
        return self.residual_history[-1]


def init_weights(init: Initialization, n1: int, n2: int) -> np.ndarray:
    """init_weights (solvers.cpp:27-38) through wgp_init_weights: cold -> zeros(n1+n2);
    warm -> [u1; 0]."""
    if n1 < 0 or n2 < 0:
        raise ValueError("init_weights: negative block size")
    if init.warm_start and init.u1.size != n1:
        raise ValueError("init_weights: warm-start vector length does not match n1")
    v = np.zeros(n1 + n2)
    u1 = np.ascontiguousarray(init.u1, dtype=np.float64) if init.warm_start else None
    _check(lib().wgp_init_weights(_ptr(u1), n1, n2, _ptr(v)))
    return v


def relative_residual(op: "KernelOperator", v, b) -> float | np.ndarray:
    """relative_residual (solvers.cpp:62-66): |H v - b| / |b| per column (zero b -> ValueError)."""
    V, B = _f64(v), _f64(b)
    one = V.ndim == 1
    V = V.reshape(op.n, -1, order="F")
    B = B.reshape(op.n, -1, order="F")
    out = np.zeros(V.shape[1])
    _check(lib().wgp_relative_residual(op._h, _ptr(V), op.n, _ptr(B), op.n, V.shape[1], _ptr(out)))
    return float(out[0]) if one else out


def quadratic_objective(op: "KernelOperator", v, b) -> float | np.ndarray:
    """quadratic_objective (solvers.cpp:68-70): 0.5 v.Hv - v.b per column."""
    V, B = _f64(v), _f64(b)
    one = V.ndim == 1
    V = V.reshape(op.n, -1, order="F")
    B = B.reshape(op.n, -1, order="F")
    out = np.zeros(V.shape[1])
    _check(lib().wgp_quadratic_objective(op._h, _ptr(V), op.n, _ptr(B), op.n, V.shape[1], _ptr(out)))
    return float(out[0]) if one else out


def cross_kernel(op: "KernelOperator", Xs) -> np.ndarray:
    """cross_kernel (kernel.cpp:74-89): dense K(X*, X_op), m x n fp64, no noise term."""
    Xs = _f64(Xs)
    m = Xs.shape[0]
    K = np.zeros((m, op.n), order="F")
    _check(lib().wgp_cross_kernel(op._h, _ptr(Xs), m, max(m, 1), _ptr(K), max(m, 1)))
    return K


class CgPreconditioner:
    """CgPreconditioner (solvers.hpp:82-100) as a device handle: built once, shared by many
    cg_solve_with calls (bo_round, thompson.cpp:359-384)."""

    def __init__(self, op: "KernelOperator", handle):
        self.op = op
        self._h = handle

    @staticmethod
    def from_matrix(op: "KernelOperator", rank: int, shift: float, mode: int = SHIFT_CALIBRATED):
        h = C.c_void_p()
        _check(lib().wgp_precond_create(op._h, int(rank), float(shift), int(mode), C.byref(h)))
        return CgPreconditioner(op, h)

    @staticmethod
    def from_factor(op: "KernelOperator", L, shift: float):
        L = _f64(L).reshape(op.n, -1, order="F")
        h = C.c_void_p()
        _check(lib().wgp_precond_create_from_factor(op._h, _ptr(L), max(op.n, 1), L.shape[1],
                                                    float(shift), C.byref(h)))
        return CgPreconditioner(op, h)

    def info(self):
        k, sh = C.c_int64(), C.c_double()
        _check(lib().wgp_precond_get(self._h, C.byref(k), C.byref(sh)))
        return k.value, sh.value

    def is_identity(self) -> bool:
        return self.info()[0] == 0

    def apply(self, r) -> np.ndarray:
        R = _f64(r)
        one = R.ndim == 1
        R = R.reshape(self.op.n, -1, order="F")
        Z = np.zeros_like(R, order="F")
        _check(lib().wgp_precond_apply(self._h, _ptr(R), self.op.n, R.shape[1], _ptr(Z), self.op.n))
        return Z[:, 0] if one else Z

    def __del__(self):
        try:
            if self._h:
                lib().wgp_precond_destroy(self._h)
                self._h = None
        except Exception:
            pass


def solve_many(op: KernelOperator, rhs, inits: list, cfg: SolverConfig, return_status: bool = False):
    """solve_many (solvers.cpp:321-354) on the device: all columns in one batched solve.

    Raises at the lowest failing column like the reference.  With
    ``return_status=True`` a DivergenceError is not raised; returns (results, status,
    diverged_at) so callers can implement solve_best_effort (thompson.cpp:299-317).  Every
    other error (NotSpdError, invalid arguments) still raises."""
    B = _f64(rhs)
    if B.ndim == 1:
        B = B.reshape(-1, 1, order="F")
    n, s = B.shape
    if len(inits) != s:
        raise ValueError("solve_many: one initialization per right-hand side required")
    if n != op.n:
        raise ValueError("solve_many: rhs rows != operator size")
    warm = [i.warm_start for i in inits]
    U1 = None
    n1 = 0
    if any(warm):
        n1s = {i.u1.size for i in inits if i.warm_start}
        if len(n1s) != 1:
            raise ValueError("solve_many: warm starts must share one length")
        n1 = n1s.pop()
        U1 = np.zeros((n1, s), order="F")
        for c, i in enumerate(inits):
            if i.warm_start:
                U1[:, c] = i.u1
    V = np.empty((n, s), order="F")  # every entry is written by the solve
    hs = cfg.max_iters + 1
    hist = np.zeros((s, hs))
    its = np.zeros(s, dtype=np.int32)
    hl = np.zeros(s, dtype=np.int32)
    cv = np.zeros(s, dtype=np.int32)
    cst = np.zeros(s, dtype=np.int32)
    dv = np.zeros(s, dtype=np.int32)
    st = lib().wgp_solve_many(op._h, C.byref(cfg), _ptr(B), n, s, _ptr(U1), max(n1, 1), n1, _ptr(V), n,
                              _ptr(its), _ptr(hist), hs, _ptr(hl), _ptr(cv), _ptr(cst), _ptr(dv))
    # each result's v is its own (contiguous) column of the Fortran-order V: no copy
    results = [SolveResult(V[:, c], int(its[c]), hist[c, : hl[c]].tolist(), bool(cv[c]))
               for c in range(s)]
    if return_status:
        # only DivergenceError is a per-column outcome (solve_best_effort catches nothing
        # else, thompson.cpp:299-317); NOT_SPD aborts the whole solve before any output is
        # written, so it raises like every other error
        if st not in (OK, DIVERGED):
            _check(st)
        return results, cst, dv
    if st != OK:
        bad = [c for c in range(s) if cst[c] != OK]
        _check(st, int(dv[bad[0]]) if bad else 0)
    return results


def solve(op: KernelOperator, b, init: Initialization, cfg: SolverConfig) -> SolveResult:
    """solve (solvers.cpp:311-319): one RHS; SGD uses cfg.seed itself (not derive_seed)."""
    b = np.ascontiguousarray(b, dtype=np.float64).ravel()
    n = op.n
    if b.size != n:
        raise ValueError("solve: rhs length != operator size")
    u1 = None if not init.warm_start else np.ascontiguousarray(init.u1, dtype=np.float64)
    n1 = 0 if u1 is None else u1.size
    v = np.zeros(n)
    hist = np.zeros(cfg.max_iters + 1)
    its, hl, cv, dv = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    st = lib().wgp_solve(op._h, C.byref(cfg), _ptr(b), _ptr(u1), n1, _ptr(v), C.byref(its), _ptr(hist),
                         C.byref(hl), C.byref(cv), C.byref(dv))
    _check(st, dv.value)
    return SolveResult(v, its.value, hist[: hl.value].tolist(), bool(cv.value))


def cg_solve_many_with(op: KernelOperator, rhs, inits: list, cfg: SolverConfig,
                       precond: CgPreconditioner) -> list:
    """cg_solve_with (solvers.cpp:142-183) for several columns with one external preconditioner."""
    B = _f64(rhs)
    if B.ndim == 1:
        B = B.reshape(-1, 1, order="F")
    n, s = B.shape
    if len(inits) != s or n != op.n:
        raise ValueError("cg_solve_with: one initialization per column, rows == operator size")
    n1 = 0
    U1 = None
    if any(i.warm_start for i in inits):
        n1 = {i.u1.size for i in inits if i.warm_start}.pop()
        U1 = np.zeros((n1, s), order="F")
        for c, i in enumerate(inits):
            if i.warm_start:
                U1[:, c] = i.u1
    V = np.empty((n, s), order="F")
    hs = cfg.max_iters + 1
    hist = np.zeros((s, hs))
    its, hl, cv = (np.zeros(s, dtype=np.int32) for _ in range(3))
    _check(lib().wgp_cg_solve_with(op._h, precond._h, C.byref(cfg), _ptr(B), n, s, _ptr(U1), max(n1, 1), n1,
                                   _ptr(V), n, _ptr(its), _ptr(hist), hs, _ptr(hl), _ptr(cv)))
    return [SolveResult(V[:, c], int(its[c]), hist[c, : hl[c]].tolist(), bool(cv[c])) for c in range(s)]


def cg_solve_with(op: KernelOperator, b, init: Initialization, cfg: SolverConfig,
                  precond: CgPreconditioner) -> SolveResult:
    """cg_solve_with (solvers.hpp:118-119): CG reusing an externally built preconditioner."""
    return cg_solve_many_with(op, np.asarray(b, dtype=np.float64).reshape(-1, 1), [init], cfg, precond)[0]


def cg_solve(op, b, init, cfg) -> SolveResult:
    return solve(op, b, init, cfg.copy(method=CG))


def sgd_solve(op, b, init, cfg) -> SolveResult:
    return solve(op, b, init, cfg.copy(method=SGD))


def ap_solve(op, b, init, cfg) -> SolveResult:
    return solve(op, b, init, cfg.copy(method=AP))


def pivoted_cholesky(op: KernelOperator, rank: int) -> np.ndarray:
    """pivoted_cholesky (solvers.cpp:72-107) on the device; returns n x achieved (column-major)."""
    n = op.n
    L = np.zeros((n, max(rank, 0)), order="F")
    ach = C.c_int64()
    _check(lib().wgp_pivoted_cholesky(op._h, rank, _ptr(L) if rank > 0 else None, max(n, 1), C.byref(ach)))
    return np.asfortranarray(L[:, : ach.value])


def precond_info(op: KernelOperator, rank: int, shift: float, mode: int = SHIFT_CALIBRATED):
    """(achieved rank, calibrated shift) of CgPreconditioner::from_matrix (solvers.cpp:123-133)."""
    ach = C.c_int64()
    sh = C.c_double()
    _check(lib().wgp_precond_info(op._h, rank, shift, mode, C.byref(ach), C.byref(sh)))
    return ach.value, sh.value


# ----------------------------------------------------------------- host randomness
_M64 = 2**64 - 1


def derive_seed(seed: int, stream: int) -> int:
    """derive_seed (rng.hpp:11-16)."""
    return int(lib().wgp_derive_seed(seed & _M64, stream & _M64))


class Rng:
    """warmgp::Rng (rng.hpp:21-61), bit-identical streams."""

    def __init__(self, seed: int):
        self._s = C.c_uint64(seed & _M64)

    def next_u64(self) -> int:
        return int(lib().wgp_rng_next_u64(C.byref(self._s)))

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = lib().wgp_rng_uniform(C.byref(self._s))
        return u if lo is None else lo + (hi - lo) * u

    def normal(self) -> float:
        return lib().wgp_rng_normal(C.byref(self._s))

    def chi_square3(self) -> float:
        return lib().wgp_rng_chi_square3(C.byref(self._s))

    def uniform_index(self, n: int) -> int:
        return int(lib().wgp_rng_uniform_index(C.byref(self._s), n))

    def derive(self, stream: int) -> "Rng":
        return Rng(derive_seed(self._s.value, stream))

    def normal_fill(self, n: int, scale: float = 1.0) -> np.ndarray:
        """n consecutive scale * normal() draws (advances this generator)."""
        out = np.zeros(n)
        lib().wgp_rng_normal_fill(C.byref(self._s), n, scale, _ptr(out))
        return out


def normal_fill(seed: int, n: int, scale: float = 1.0) -> np.ndarray:
    out = np.zeros(n)
    lib().wgp_normal_fill(seed & _M64, n, scale, _ptr(out))
    return out


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


def sample_prior(hyp: KernelHyperparams, dim: int, num_features: int, seed: int) -> RffPrior:
    """sample_prior (sampling.cpp:14-35) with the reference's RNG consumption order."""
    if not (hyp.lengthscale > 0 and hyp.signal_scale > 0 and hyp.noise_scale > 0):
        raise ValueError("kernel hyperparameters must be strictly positive")
    if dim < 1 or num_features < 1:
        raise ValueError("sample_prior: dim and num_features must be positive")
    Om = np.zeros((num_features, dim), order="F")
    ph = np.zeros(num_features)
    am = np.zeros(num_features)
    _check(lib().wgp_sample_prior(hyp.kind, hyp.lengthscale, dim, num_features, seed & _M64,
                                  _ptr(Om), _ptr(ph), _ptr(am)))
    return RffPrior(Om, ph, am, hyp.signal_scale)


def rff_eval(op: KernelOperator, priors: list, Xs=None, fast: bool = False) -> np.ndarray:
    """eval_prior (sampling.cpp:37-46) for several priors sharing F and signal scale, fused on
    the device; evaluated at the operator's rows (Xs=None) or at host points Xs (m x d)."""
    if not priors:
        return np.zeros((op.n if Xs is None else np.asarray(Xs).shape[0], 0), order="F")
    F = priors[0].num_features
    sf = priors[0].signal_scale
    for p in priors:
        if p.num_features != F or p.signal_scale != sf or p.dim != op.dim:
            raise ValueError("rff_eval: priors must share F, signal scale and the operator's dim")
    S = len(priors)
    Om = np.ascontiguousarray(np.stack([np.asfortranarray(p.frequencies).ravel(order="F") for p in priors]))
    ph = np.ascontiguousarray(np.stack([p.phases for p in priors]))
    am = np.ascontiguousarray(np.stack([p.amplitudes for p in priors]))
    if Xs is not None:
        Xs = _f64(Xs)
        if Xs.shape[1] != op.dim:
            raise ValueError("eval_prior: dimension mismatch")
        m = Xs.shape[0]
    else:
        m = op.n
    out = np.zeros((m, S), order="F")
    fn = lib().wgp_rff_eval_fast if fast else lib().wgp_rff_eval
    _check(fn(op._h, _ptr(Om), _ptr(ph), _ptr(am), F, S, sf, _ptr(Xs), m, max(m, 1), _ptr(out), max(m, 1)))
    return out


def build_sample_rhs(op: KernelOperator, prior: RffPrior, noise_scale: float, seed: int) -> np.ndarray:
    """build_sample_rhs (sampling.cpp:56-64) through wgp_build_sample_rhs: the prior at the
    operator's rows + noise_scale Rng(seed).normal() per row."""
    Om = np.asfortranarray(prior.frequencies, dtype=np.float64)
    ph = np.ascontiguousarray(prior.phases, dtype=np.float64)
    am = np.ascontiguousarray(prior.amplitudes, dtype=np.float64)
    out = np.zeros(op.n)
    _check(lib().wgp_build_sample_rhs(op._h, _ptr(Om), _ptr(ph), _ptr(am), Om.shape[0],
                                      float(prior.signal_scale), float(noise_scale), seed & _M64, _ptr(out)))
    return out


def kernel_timer_enable(on: bool = True) -> None:
    """Start (and clear) / stop CUDA-event timing of the tensor-core kmatvec kernel launches."""
    lib().wgp_kernel_timer_enable(1 if on else 0)


def kernel_timer_read(tag: str = "kmatvec_tc") -> tuple[float, int]:
    """(summed kernel milliseconds, launches) of one kernel family ("kmatvec_tc",
    "kmatvec_f64", "kmatvec_f32", "krows", "kcols", "rff_eval", "rff_eval32") since the
    last kernel_timer_enable(True)."""
    ms = C.c_double(0.0)
    n = C.c_int64(0)
    _check(lib().wgp_kernel_timer_read_tag(tag.encode(), C.byref(ms), C.byref(n)))
    return ms.value, n.value


def eval_posterior(op: KernelOperator, priors: list, weights, Xs, fast: bool = False) -> np.ndarray:
    """eval_posterior (sampling.cpp:66-75) for S pathwise samples at once: prior_s(X*) +
    K(X*, X) weights[:, s], with the operator's rows as the training inputs -> m x S."""
    weights = np.asarray(weights, dtype=np.float64)
    if weights.ndim == 1:
        weights = weights[:, None]
    if weights.shape != (op.n, len(priors)):
        raise ValueError("eval_posterior: weights length != training rows")
    out = rff_eval(op, priors, Xs, fast=fast)
    if op.n > 0:
        out = out + op.cross_matvec(Xs, weights)
    return out


def exact_solve(op: KernelOperator, b) -> np.ndarray:
    """exact_solve (analysis.cpp:15-26): H^{-1} b by a dense fp64 device Cholesky of the
    operator's H; b: n or n x s.  NotSpdError if the factorization fails."""
    B = np.asfortranarray(np.asarray(b, dtype=np.float64))
    vec = B.ndim == 1
    if vec:
        B = B.reshape(-1, 1, order="F")
    n, s = B.shape
    Xo = np.zeros((n, s), order="F")
    _check(lib().wgp_exact_solve(op._h, _ptr(B), n, s, _ptr(Xo), n))
    return Xo[:, 0] if vec else Xo


@dataclass
class MllResult:
    """warmgp::MllResult (analysis.hpp:42-45): value and d/d(log l, log s_f, log sigma_n)."""
    value: float
    grad: np.ndarray


def _mll_op(X_or_op, hyp):
    if isinstance(X_or_op, KernelOperator):
        return X_or_op
    if hyp is None:
        raise ValueError("mll: hyperparameters required with raw inputs")
    return KernelOperator(hyp, X_or_op, precision=F64)


def mll(X_or_op, y, hyp: KernelHyperparams | None = None) -> MllResult:
    """mll (analysis.cpp:99-139) on the device: X_or_op is the inputs (n x d; a temporary fp64
    operator is built) or an operator (its rows); hyp defaults to the operator's.  Matern-3/2
    as the reference (RBF analogue for RBF operators).  NotSpdError if H is not SPD."""
    op = _mll_op(X_or_op, hyp)
    y = np.ascontiguousarray(np.asarray(y, dtype=np.float64).ravel())
    if y.shape[0] != op.n:
        raise ValueError("mll: X rows != y length")
    h3 = None if hyp is None else np.array([hyp.lengthscale, hyp.signal_scale, hyp.noise_scale])
    val = C.c_double(0.0)
    g = np.zeros(3)
    _check(lib().wgp_mll(op._h, _ptr(y), _ptr(h3), C.byref(val), _ptr(g)))
    return MllResult(val.value, g)


def optimize_mll(X_or_op, y, init_hyp: KernelHyperparams, steps: int, step_size: float) -> KernelHyperparams:
    """optimize_mll (analysis.cpp:141-182): Adam on the log-parameters (device MLL per step);
    returns the best hyperparameters seen.  RuntimeError on a non-finite MLL."""
    op = _mll_op(X_or_op, init_hyp)
    y = np.ascontiguousarray(np.asarray(y, dtype=np.float64).ravel())
    if y.shape[0] != op.n:
        raise ValueError("optimize_mll: X rows != y length")
    h3 = np.array([init_hyp.lengthscale, init_hyp.signal_scale, init_hyp.noise_scale])
    out = np.zeros(3)
    _check(lib().wgp_optimize_mll(op._h, _ptr(y), _ptr(h3), int(steps), float(step_size), _ptr(out)))
    return KernelHyperparams(float(out[0]), float(out[1]), float(out[2]), init_hyp.kind)


def median_heuristic_lengthscale(X, seed: int = 0) -> float:
    """median_heuristic_lengthscale (analysis.cpp:184-203)."""
    X = _f64(X)
    return float(lib().wgp_median_heuristic_lengthscale(_ptr(X), X.shape[0], max(X.shape[0], 1), X.shape[1],
                                                        seed & (2**64 - 1)))


def _stack_priors(priors):
    F = priors[0].num_features
    sf = priors[0].signal_scale
    for p in priors:
        if p.num_features != F or p.signal_scale != sf:
            raise ValueError("priors must share F and the signal scale")
    Om = np.ascontiguousarray(np.stack([np.asfortranarray(p.frequencies).ravel(order="F") for p in priors]))
    ph = np.ascontiguousarray(np.stack([p.phases for p in priors]))
    am = np.ascontiguousarray(np.stack([p.amplitudes for p in priors]))
    return Om, ph, am, F, sf


def posterior_select(op: KernelOperator, priors: list, weights, Xs, groups: int = 1,
                     fast: bool = True) -> np.ndarray:
    """select_peaks' argmax (thompson.cpp:199-203) on the device: for every sample s and
    contiguous candidate group g, the first candidate row with the largest posterior value
    prior_s(X*) + K(X*, X) weights[:, s].  Returns S x groups int64 row indices."""
    Om, ph, am, F, sf = _stack_priors(priors)
    S = len(priors)
    Wt = np.asfortranarray(weights, dtype=np.float64).reshape(op.n, S, order="F")
    Xs = _f64(Xs)
    m = Xs.shape[0]
    idx = np.zeros((S, groups), dtype=np.int64)
    _check(lib().wgp_posterior_select(op._h, _ptr(Om), _ptr(ph), _ptr(am), F, S, sf, _ptr(Wt), op.n,
                                      _ptr(Xs), m, m, int(groups), 1 if fast else 0, _ptr(idx)))
    return idx


def grad_posterior(op: KernelOperator, priors: list, weights, Xs, sample_index) -> np.ndarray:
    """grad_posterior (sampling.cpp:77-87) at m points; point i uses sample sample_index[i]
    (prior priors[s], weights[:, s]) with the operator's rows as training inputs -> m x dim."""
    Om, ph, am, F, sf = _stack_priors(priors)
    Wt = np.asfortranarray(np.asarray(weights, dtype=np.float64).reshape(op.n, len(priors)))
    Xs = np.asfortranarray(np.asarray(Xs, dtype=np.float64))
    m = Xs.shape[0]
    sidx = np.ascontiguousarray(np.asarray(sample_index, dtype=np.int32))
    G = np.zeros((m, op.dim), order="F")
    _check(lib().wgp_grad_posterior(op._h, _ptr(Om), _ptr(ph), _ptr(am), F, len(priors), sf, _ptr(Wt),
                                    max(op.n, 1), _ptr(Xs), max(m, 1), _ptr(sidx), m, _ptr(G), max(m, 1)))
    return G


def ascend_peaks(op: KernelOperator, priors: list, weights, starts, steps: int, rate: float):
    """ascend_peaks (thompson.cpp:209-258) for all samples at once; starts: S x P x dim.
    Returns (best points S x dim, best values S)."""
    Om, ph, am, F, sf = _stack_priors(priors)
    S = len(priors)
    starts = np.asarray(starts, dtype=np.float64)
    P = starts.shape[1]
    Wt = np.asfortranarray(np.asarray(weights, dtype=np.float64).reshape(op.n, S))
    st = np.asfortranarray(starts.reshape(S * P, op.dim))
    bx = np.zeros((S, op.dim), order="F")
    bv = np.zeros(S)
    _check(lib().wgp_ascend_peaks(op._h, _ptr(Om), _ptr(ph), _ptr(am), F, S, sf, _ptr(Wt), max(op.n, 1),
                                  _ptr(st), P, steps, rate, _ptr(bx), _ptr(bv)))
    return bx, bv

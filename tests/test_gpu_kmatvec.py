"""GPU parity of the fused kernel-matvec (K1) against the CPU oracle, through the C-ABI.

Bars (BASELINE.json north_star): relative error <= 1e-10 on the fp64 path and
<= 1e-4 on the fp32/tf32 path, measured per RHS column as |Y - Y_ref| / |Y_ref|.
"""
import glob
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = {0: 1e-10, 1: 1e-4, 3: 1e-4}  # F64, F32_3XTF32, F32_SIMT


def colrel(Y, Yref):
    return float(np.max(np.linalg.norm(Y - Yref, axis=0) / np.linalg.norm(Yref, axis=0)))


def hyp_of(W, arr):
    kind, ls, sf, sn = arr
    return W.KernelHyperparams(float(ls), float(sf), float(sn), int(kind))


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(HERE, "golden", "kmatvec_*.npz"))),
                         ids=lambda p: os.path.basename(p)[8:-4])
@pytest.mark.parametrize("precision", [0, 1, 3])
def test_kmatvec_golden(W, path, precision):
    g = np.load(path)
    op = W.KernelOperator(hyp_of(W, g["hyp"]), g["X"], precision=precision)
    Y = op.kmatvec(g["V"])
    assert colrel(Y, g["Y"]) <= TOL[precision]


@pytest.mark.parametrize("n,d,s", [(1, 3, 1), (2, 1, 2), (63, 5, 3), (65, 16, 17), (200, 8, 129), (1000, 2, 64)])
@pytest.mark.parametrize("kind", [0, 1])
def test_kmatvec_shapes_vs_oracle(W, O, n, d, s, kind):
    h = O.KernelHyperparams(0.6, 1.3, 0.2, kind)
    X = O.uniform_inputs(n * 7 + d, n, d)
    V = np.random.default_rng(n + s).standard_normal((n, s))
    Yref = O.kmatvec(X, h, V)
    for prec in (0, 1, 3):
        op = W.KernelOperator(W.KernelHyperparams(0.6, 1.3, 0.2, kind), X, precision=prec)
        assert colrel(op.kmatvec(V), Yref) <= TOL[prec], prec


def test_append_rows_equals_concat(W, O):
    h = O.KernelHyperparams(0.5, 1.0, 0.1, O.MATERN32)
    X1 = O.uniform_inputs(51, 300, 3)
    X2 = O.uniform_inputs(52, 700, 3)
    X = np.vstack([X1, X2])
    V = np.random.default_rng(0).standard_normal((1000, 4))
    op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1, 0), X1)
    op.append_rows(X2[:100])
    op.append_rows(X2[100:])  # crosses the initial capacity (1024 rows) growth path
    assert op.n == 1000
    assert colrel(op.kmatvec(V), O.kmatvec(X, h, V)) <= 1e-12


def test_cross_matvec_vs_oracle(W, O):
    h = O.KernelHyperparams(0.3, 1.1, 1e-3, O.MATERN32)
    X = O.uniform_inputs(61, 400, 4)
    Xs = O.uniform_inputs(62, 333, 4)
    Wt = np.random.default_rng(1).standard_normal((400, 5))
    ref = O.cross_kernel(Xs, X, h) @ Wt
    for prec in (0, 1):
        op = W.KernelOperator(W.KernelHyperparams(0.3, 1.1, 1e-3, 0), X, precision=prec)
        assert colrel(op.cross_matvec(Xs, Wt), ref) <= TOL[prec]


def test_cross_matvec_tensor_core_path(W):
    """Cross mode K(X*, X) W on the tensor cores (posterior evaluation at candidates, SURVEY
    8f.1): wide RHS (two column chunks), ragged sizes, against the fp64 operator; points far
    outside the fp16 operand range take the fp64 fallback and stay exact."""
    rng = np.random.default_rng(7)
    X = rng.random((3001, 5))
    Xs = rng.random((4999, 5))
    Wt = rng.standard_normal((3001, 70))
    for kind, ls in ((0, 0.3), (1, 0.5)):
        h = W.KernelHyperparams(ls, 1.3, 0.1, kind)
        ref = W.KernelOperator(h, X, precision=W.F64).cross_matvec(Xs, Wt)
        got = W.KernelOperator(h, X, precision=W.F32_3XTF32).cross_matvec(Xs, Wt)
        assert colrel(got, ref) <= 1e-5
        far = Xs[:50] + 1e3  # |x - c| / l >> 64: no fp16 operands for these rows
        ref_far = W.KernelOperator(h, X, precision=W.F64).cross_matvec(far, Wt)
        got_far = W.KernelOperator(h, X, precision=W.F32_3XTF32).cross_matvec(far, Wt)
        assert np.array_equal(got_far, ref_far)


def test_kmatvec_linearity_large(W):
    """Size-independent property at a BASELINE-scale N: H(aU + bV) = aHU + bHV."""
    rng = np.random.default_rng(5)
    n, d = 20000, 8
    X = rng.random((n, d))
    U = rng.standard_normal((n, 4))
    V = rng.standard_normal((n, 4))
    op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1, 1), X, precision=1)
    lhs = op.kmatvec(2.0 * U - 3.0 * V)
    rhs = 2.0 * op.kmatvec(U) - 3.0 * op.kmatvec(V)
    assert colrel(lhs, rhs) <= 1e-4


def test_invalid_arguments(W):
    with pytest.raises(ValueError):
        W.KernelOperator(W.KernelHyperparams(-1.0, 1.0, 0.1), np.zeros((3, 2)))
    op = W.KernelOperator(W.KernelHyperparams(1.0, 1.0, 0.1), np.zeros((3, 2)))
    with pytest.raises(ValueError):
        op.append_rows(np.zeros((2, 3)))
    with pytest.raises(ValueError):
        op.kmatvec(np.zeros((4, 1)))


@pytest.mark.parametrize("n", [20000, 101000])
def test_tc_accuracy_scales_with_n(W, n):
    """Size-independent cross-check at BASELINE scale: the tensor-core path against the fp64
    CUDA-core path (itself pinned to the oracle at <=1e-10 above), relative error <= 1e-4."""
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, 16))
    V = rng.standard_normal((n, 4))
    hyp = W.KernelHyperparams(0.8, 1.0, 1e-3 ** 0.5, 0)
    Y64 = W.KernelOperator(hyp, X, precision=W.F64).kmatvec(V)
    Ytc = W.KernelOperator(hyp, X, precision=W.F32_3XTF32).kmatvec(V)
    err = colrel(Ytc, Y64)
    print(f"n={n} tc rel err {err:.3e}")
    assert err <= 1e-4


def test_kernel_timer_counts_tc_launches(W):
    """wgp_kernel_timer_*: CUDA-event timing of the tensor-core kernel launches only (bench.py's
    roofline numerator); one launch per 64-column RHS chunk, and the host API splits a single
    chunk's rows in four launches (each part's copy-back overlaps the next parts)."""
    rng = np.random.default_rng(3)
    X = rng.random((5000, 6))
    op = W.KernelOperator(W.KernelHyperparams(0.4, 1.0, 0.1, 0), X, precision=W.F32_3XTF32)
    V = rng.standard_normal((5000, 100))
    W.kernel_timer_enable(True)
    op.kmatvec(V)
    op.kmatvec(V[:, :10])
    ms, n = W.kernel_timer_read()
    W.kernel_timer_enable(False)
    assert n == 2 + 4 and ms > 0.0
    W.kernel_timer_enable(False)
    op.kmatvec(V[:, :10])
    assert W.kernel_timer_read() == (0.0, 0)


@pytest.mark.parametrize("d", [24, 32])
def test_tc_wide_dims_and_tf32_operand_fallback(W, d):
    """Tensor-core path at the widest supported dims, and with coordinates far outside the fp16
    operand range (|x|/l >> 64), which switches GEMM1 to tf32 operands: both stay within the
    fp32 bar of the fp64 operator."""
    rng = np.random.default_rng(d)
    X = rng.random((3000, d))
    V = rng.standard_normal((3000, 8))
    for scale, ls in ((1.0, 0.9), (300.0, 0.9 * 300.0 / 5.0)):
        Xs = X * scale
        h = W.KernelHyperparams(ls, 1.0, 0.1, W.MATERN32)
        ref = W.KernelOperator(h, Xs, precision=W.F64).kmatvec(V)
        got = W.KernelOperator(h, Xs, precision=W.F32_3XTF32).kmatvec(V)
        assert colrel(got, ref) <= 1e-4, (d, scale)


def test_tf32_precision_mode(W):
    """WGP_TF32: single-pass tf32 distances (not parity-grade): ~1e-3, documented."""
    rng = np.random.default_rng(11)
    X = rng.random((4000, 6))
    V = rng.standard_normal((4000, 16))
    h = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
    ref = W.KernelOperator(h, X, precision=W.F64).kmatvec(V)
    got = W.KernelOperator(h, X, precision=W.TF32).kmatvec(V)
    assert colrel(got, ref) <= 5e-3


@pytest.mark.parametrize("n,s", [(130, 3), (700, 64), (9000, 17), (33001, 100)])
def test_tc_split_grids(W, n, s):
    """Grid shapes from a single CTA (n = 130) through several j-splits per row block (n = 9000,
    33001) and a ragged two-chunk RHS (s = 100): every split's partial slot is written and the
    reduction adds them -- checked against the fp64 operator, diagonal included."""
    rng = np.random.default_rng(n)
    X = rng.random((n, 7))
    V = rng.standard_normal((n, s))
    for kind in (0, 1):
        h = W.KernelHyperparams(0.4, 1.1, 0.05, kind)
        ref = W.KernelOperator(h, X, precision=W.F64).kmatvec(V)
        got = W.KernelOperator(h, X, precision=W.F32_3XTF32).kmatvec(V)
        assert colrel(got, ref) <= 2e-5, (n, s, kind)


@pytest.mark.parametrize("s", [17, 129])
def test_f64_column_splits_batch_independent(W, O, s):
    """fp64 kernel-matvec past one 4096-column split (n = 9000: three splits summed in order):
    each column equals its single-column product bitwise (the batched-vs-sequential contract of
    solve_many, test_solvers.cpp:397-413) and matches the oracle at the fp64 bar."""
    n = 9000
    X = O.uniform_inputs(77, n, 3)
    V = np.random.default_rng(s).standard_normal((n, s))
    h = O.KernelHyperparams(0.3, 1.0, 0.1, O.MATERN32)
    op = W.KernelOperator(W.KernelHyperparams(0.3, 1.0, 0.1, W.MATERN32), X, precision=W.F64)
    Y = op.kmatvec(V)
    for c in (0, s // 2, s - 1):
        assert np.array_equal(Y[:, c], op.kmatvec(V[:, c:c + 1])[:, 0]), c
    ref = O.kmatvec(X, h, V[:, :3])
    assert colrel(Y[:, :3], ref) <= 1e-10


@pytest.mark.parametrize("kind,n,d,s", [(0, 30_000, 16, 64), (1, 20_000, 8, 17), (0, 3_000, 6, 129)])
def test_tc_kernel_repeat_launches_bitwise(W, kind, n, d, s):
    """Race check of the tcgen05 pipeline (28 warps, mbarrier rings over smem and TMEM,
    in-place TMEM overwrite of S by K) by repetition: compute-sanitizer is not available on
    this GPU pool, so every launch of the same input must give bitwise the same output (a
    producer/consumer race on a ring slot or a TMEM buffer would show up as occasional
    differences; the partial-sum order is fixed per thread, so the kernel is deterministic
    by construction)."""
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, d)) if kind == 0 else rng.random((n, d))
    V = np.asfortranarray(rng.standard_normal((n, s)))
    op = W.KernelOperator(W.KernelHyperparams(0.8, 1.0, 0.05, kind), X, precision=W.F32_3XTF32)
    ref = op.kmatvec(V)
    for _ in range(12):
        assert np.array_equal(op.kmatvec(V), ref)


@pytest.mark.parametrize("kind,n,d,s", [(0, 40_003, 16, 64), (1, 20_000, 8, 5)])
def test_host_form_column_parts(W, kind, n, d, s):
    """The host-buffer matvec on a tensor-core operator uploads V in three column parts and
    computes each part's columns as it lands (the diagonal and sigma^2 V_i once, in the right
    parts), the last part in four row parts: it agrees with the device form (one launch over
    all columns) to fp32-accumulation rounding, with the fp64 operator at the fp32 bar, and is
    deterministic.  Kernel launches: one per leading column part, four for the last."""
    import torch
    rng = np.random.default_rng(n + s)
    X = rng.standard_normal((n, d)) if kind == 0 else rng.random((n, d))
    V = np.asfortranarray(rng.standard_normal((n, s)))
    h = W.KernelHyperparams(0.8, 1.0, 0.05, kind)
    op = W.KernelOperator(h, X, precision=W.F32_3XTF32)
    W.kernel_timer_enable(True)
    Y = op.kmatvec(V)
    _, launches = W.kernel_timer_read()
    W.kernel_timer_enable(False)
    assert launches == 2 + 4
    Vd = torch.from_numpy(np.ascontiguousarray(V)).cuda()
    Yd = torch.empty_like(Vd)
    op.kmatvec_dev(Vd.data_ptr(), Yd.data_ptr(), s)
    torch.cuda.synchronize()
    assert colrel(Y, Yd.cpu().numpy()) <= 5e-6
    ref = W.KernelOperator(h, X, precision=W.F64).kmatvec(V)
    assert colrel(Y, ref) <= 1e-4
    assert np.array_equal(op.kmatvec(V), Y)


_TILE_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2511_16340_b200 import warmgp as W
rng = np.random.default_rng(11)
out = []
for kind, n, d, s in ((1, 3000, 8, 32), (0, 2500, 16, 17), (1, 1700, 5, 4)):
    X = rng.random((n, d)) * 2.0
    V = rng.standard_normal((n, s))
    op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1, kind), X, precision=W.F32_3XTF32)
    out.append(op.kmatvec(V))
np.savez({path!r}, *out)
"""


@pytest.mark.parametrize("bj", ["64", "128"])
def test_tc_tile_widths_agree(W, O, bj, tmp_path):
    """Both tile widths of the tensor-core kernel (WGP_TC_BJ, read once per process: each in
    its own child process) give the oracle's product within the fp32 bar at s <= 32, where
    the default is the 128-column tile with three TMEM buffers."""
    import subprocess
    import sys

    root = os.path.dirname(HERE)
    path = str(tmp_path / f"y{bj}.npz")
    env = dict(os.environ, WGP_TC_BJ=bj)
    subprocess.run([sys.executable, "-c", _TILE_CHILD.format(root=root, path=path)], env=env, check=True,
                   timeout=300)
    got = np.load(path)
    rng = np.random.default_rng(11)
    for k, (kind, n, d, s) in enumerate(((1, 3000, 8, 32), (0, 2500, 16, 17), (1, 1700, 5, 4))):
        X = rng.random((n, d)) * 2.0
        V = rng.standard_normal((n, s))
        ref = O.kmatvec(X, O.KernelHyperparams(0.5, 1.0, 0.1, kind), np.asfortranarray(V))
        assert colrel(got[f"arr_{k}"], ref) <= 1e-5, (bj, kind, n, d, s)


@pytest.mark.parametrize("kind", [0, 1])
def test_tc_far_pairs_underflow_cleanly(W, O, kind):
    """Pairs far beyond the kernel's range (exponent arguments below the FMA-pipe exp2's
    -100 clamp and below fp16's range after the 2^10 scale) contribute zeros: a few points
    ~40 lengthscales from the rest (z ~ 140 for Matern, d^2/2l^2 ~ 3000 for RBF) give no
    NaN/Inf and the oracle's product within the fp32 bar."""
    rng = np.random.default_rng(3)
    n, d, s = 1500, 4, 8
    X = rng.random((n, d))
    X[-10:] += 10.0  # 20 units per coordinate = 40 lengthscales away (|x - c| / l < 64 still)
    V = rng.standard_normal((n, s))
    h = O.KernelHyperparams(0.5, 1.0, 0.1, kind)
    op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.1, kind), X, precision=W.F32_3XTF32)
    Y = op.kmatvec(V)
    assert np.all(np.isfinite(Y))
    ref = O.kmatvec(X, h, np.asfortranarray(V))
    assert colrel(Y, ref) <= 1e-4

"""GPU checks of the fused solver vector kernels (north-star item 2) through the C-ABI
device entry points: v += alpha p (solvers.cpp:168), p = z + beta p (:180) and the column
dot products p.Hp / |r|^2 / r.z (:163,172,179).

The element-wise updates are compared with numpy (same fp64 expression; at most one
rounding of difference where the compiler contracts to an FMA).  The dot products are
compared with an exact restatement of the fixed summation order (512-row chunks, 32
sequential 16-row slabs each, slabs then chunks added in index order) and checked to be
bitwise independent of the number of columns s -- the property that makes solve_many equal
sequential single solves (test_solvers.cpp:397-413) and sharded runs equal unsharded ones.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(W):
    import torch

    ctx = W.DeviceContext(0)
    yield ctx, torch
    ctx.close()


def ordered_coldots(A, B):
    """The device's summation order, restated in fp64."""
    n, s = A.shape
    out = np.zeros(s)
    for c in range(s):
        tot = 0.0
        for c0 in range(0, n, 512):
            chunk = 0.0
            for q in range(32):
                i0 = c0 + 16 * q
                acc = 0.0
                for i in range(i0, min(n, i0 + 16)):
                    acc = acc + A[i, c] * B[i, c]  # the device fuses this into one fma
                chunk += acc
            tot += chunk
        out[c] = tot
    return out


@pytest.mark.parametrize("n,s", [(1, 1), (17, 3), (1000, 17), (5000, 64), (101000, 64)])
def test_axpy_xpby(dev, n, s):
    ctx, torch = dev
    rng = np.random.default_rng(n + s)
    Y0, X0 = rng.standard_normal((n, s)), rng.standard_normal((n, s))
    alpha = rng.standard_normal(s)
    alpha[0] = 0.0  # frozen column: untouched
    active = (rng.random(s) > 0.3).astype(np.int32)
    Y, X = torch.tensor(Y0, device="cuda"), torch.tensor(X0, device="cuda")
    a = torch.tensor(alpha, device="cuda")
    torch.cuda.synchronize()  # inputs are made on torch's stream, the op runs on the context's
    ctx.axpy_cols_dev(Y.data_ptr(), X.data_ptr(), a.data_ptr(), n, s)
    torch.cuda.synchronize()
    ref = Y0 + alpha * X0
    got = Y.cpu().numpy()
    assert np.array_equal(got[:, 0], Y0[:, 0])
    np.testing.assert_allclose(got, ref, rtol=1e-15, atol=1e-15 * np.abs(alpha * X0).max())

    P0 = rng.standard_normal((n, s))
    P, act = torch.tensor(P0, device="cuda"), torch.tensor(active, device="cuda")
    torch.cuda.synchronize()
    ctx.xpby_cols_dev(P.data_ptr(), X.data_ptr(), a.data_ptr(), act.data_ptr(), n, s)
    torch.cuda.synchronize()
    got = P.cpu().numpy()
    ref = np.where(active.astype(bool), X0 + alpha * P0, P0)
    assert np.array_equal(got[:, active == 0], P0[:, active == 0])
    np.testing.assert_allclose(got, ref, rtol=1e-15, atol=1e-15 * np.abs(alpha * P0).max())


@pytest.mark.parametrize("n,s", [(1, 1), (15, 2), (513, 3), (3001, 9)])
def test_coldots_order(dev, n, s):
    ctx, torch = dev
    rng = np.random.default_rng(7 * n + s)
    A0, B0 = rng.standard_normal((n, s)), rng.standard_normal((n, s))
    A, B = torch.tensor(A0, device="cuda"), torch.tensor(B0, device="cuda")
    out = torch.empty(s, device="cuda", dtype=torch.float64)
    work = torch.empty(((n + 511) // 512) * s, device="cuda", dtype=torch.float64)
    torch.cuda.synchronize()
    ctx.coldots_dev(A.data_ptr(), B.data_ptr(), n, s, out.data_ptr(), work.data_ptr())
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    ref = ordered_coldots(A0, B0)
    np.testing.assert_allclose(got, ref, rtol=1e-14, atol=1e-14 * np.sqrt(n))
    np.testing.assert_allclose(got, np.einsum("ic,ic->c", A0, B0), rtol=1e-12, atol=1e-12 * np.sqrt(n))


def test_coldots_column_independent(dev):
    """A column's dot product is bitwise the same whatever the other columns are."""
    ctx, torch = dev
    n, s = 101000, 64
    rng = np.random.default_rng(3)
    A0, B0 = rng.standard_normal((n, s)), rng.standard_normal((n, s))
    A, B = torch.tensor(A0, device="cuda"), torch.tensor(B0, device="cuda")
    work = torch.empty(((n + 511) // 512) * s, device="cuda", dtype=torch.float64)
    full = torch.empty(s, device="cuda", dtype=torch.float64)
    torch.cuda.synchronize()
    ctx.coldots_dev(A.data_ptr(), B.data_ptr(), n, s, full.data_ptr(), work.data_ptr())
    torch.cuda.synchronize()
    for c in (0, 17, 63):
        a1 = A[:, c].contiguous()
        b1 = B[:, c].contiguous()
        one = torch.empty(1, device="cuda", dtype=torch.float64)
        torch.cuda.synchronize()
        ctx.coldots_dev(a1.data_ptr(), b1.data_ptr(), n, 1, one.data_ptr(), work.data_ptr())
        torch.cuda.synchronize()
        assert one.item() == full[c].item()
    np.testing.assert_allclose(full.cpu().numpy(), np.einsum("ic,ic->c", A0, B0), rtol=1e-11)


def test_vecops_bad_arguments(dev, W):
    ctx, torch = dev
    with pytest.raises(ValueError):
        ctx.coldots_dev(0, 0, 10, 1, 0, 0)

"""The device block cache behind every library buffer (csrc/mem.cpp): blocks carved from
shared chunks and recycled by size bucket must never overlap while alive.  Many operators of
different sizes and precisions live at once, are destroyed in a scrambled order and recreated,
and every product is checked against the same product computed by a fresh operator at the
end (bitwise: the kernels are deterministic)."""
import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_block_cache_no_overlap_bitwise(W):
    rng = np.random.default_rng(123)
    shapes = [(300, 3, 5, W.F64), (1000, 8, 17, W.F32_3XTF32), (4097, 16, 33, W.F32_3XTF32),
              (2500, 5, 64, W.F64), (700, 2, 1, W.F32_3XTF32), (6000, 8, 32, W.F32_3XTF32)]
    inputs = []
    for n, d, s, prec in shapes:
        X = rng.random((n, d))
        V = rng.standard_normal((n, s))
        kind = W.RBF if d % 2 == 0 else W.MATERN32
        inputs.append((X, V, W.KernelHyperparams(0.6, 1.1, 0.2, kind), prec))
    ops = [W.KernelOperator(h, X, precision=p) for X, V, h, p in inputs]
    first = [op.kmatvec(V) for op, (X, V, h, p) in zip(ops, inputs)]
    # interleave: destroy half, grow others, recompute, recreate
    for k in (3, 0, 5):
        ops[k] = None
    gc.collect()
    again = {k: ops[k].kmatvec(inputs[k][1]) for k in (1, 2, 4)}
    for k in (1, 2, 4):
        assert np.array_equal(again[k], first[k]), k
    for k in (3, 0, 5):
        X, V, h, p = inputs[k]
        ops[k] = W.KernelOperator(h, X, precision=p)
    last = [op.kmatvec(V) for op, (X, V, h, p) in zip(ops, inputs)]
    for k in range(len(shapes)):
        assert np.array_equal(last[k], first[k]), k
    # solves keep their workspaces on the operator: two solves on one operator, a third on a
    # fresh one, identical results
    X, V, h, p = inputs[1]
    cfg = W.SolverConfig(tolerance=1e-6, max_iters=300, precond_rank=20, precond_shift=0.04)
    inits = [W.Initialization.cold()] * V.shape[1]
    a = W.solve_many(ops[1], V, inits, cfg)
    b = W.solve_many(ops[1], V, inits, cfg)
    c = W.solve_many(W.KernelOperator(h, X, precision=p), V, inits, cfg)
    for ra, rb, rc in zip(a, b, c):
        assert np.array_equal(ra.v, rb.v) and np.array_equal(ra.v, rc.v)
        assert ra.iterations == rb.iterations == rc.iterations

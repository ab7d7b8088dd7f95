"""world_size-2 CPU (gloo) test of the row-sharded CG decomposition:
rows partitioned by wgp_shard_range, per-column dot products as fixed 512-row chunk
partials all-gathered and summed in chunk order, direction/solution slices all-gathered
before each operator application.  The sharded run must reproduce the single-process
run bit for bit (iteration counts and histories), which is what makes the CUDA/NCCL
path's results independent of the GPU count."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CHUNK = 512


def shard_range(n, world, rank):
    """Equal slots of ceil(nch / world) chunks (wgp_shard_range; the exchange is one
    in-place all-gather of equal slices of a buffer padded to world slots)."""
    nch = (n + CHUNK - 1) // CHUNK
    c = max(1, -(-nch // world))
    return min(rank * c * CHUNK, n), min((rank + 1) * c * CHUNK, n)


def chunk_dots(a, b, row0):
    """Partials of sum(a*b) per global chunk over this rank's rows (a, b: local rows)."""
    out = {}
    for lo in range(0, a.shape[0], CHUNK):
        c = (row0 + lo) // CHUNK
        out[c] = float(np.dot(a[lo:lo + CHUNK], b[lo:lo + CHUNK]))
    return out


def gather_sum(parts, world):
    if world == 1:
        allp = [parts]
    else:
        allp = [None] * world
        dist.all_gather_object(allp, parts)
    merged = {}
    for d in allp:
        merged.update(d)
    return sum(merged[c] for c in sorted(merged))  # fixed chunk order


def gather_rows(local, n, world):
    if world == 1:
        return local.copy()
    pieces = [None] * world
    dist.all_gather_object(pieces, local)
    return np.concatenate(pieces)


def rowdot(Hl, v):
    """Per-row dot products: each row's summation order is independent of how many rows a
    rank holds (as in the CUDA kernel-matvec, where a row's j-tile order is fixed)."""
    return np.array([np.dot(row, v) for row in Hl])


def sharded_cg(H, b, rank, world, tol=1e-8, max_iters=200):
    n = b.size
    r0, r1 = shard_range(n, world, rank)
    Hl = H[r0:r1]
    bl = b[r0:r1]
    v = np.zeros(n)
    bnorm = np.sqrt(gather_sum(chunk_dots(bl, bl, r0), world))
    r = bl - rowdot(Hl, v)
    hist = [np.sqrt(gather_sum(chunk_dots(r, r, r0), world)) / bnorm]
    z = r.copy()
    p_l = z.copy()
    rz = gather_sum(chunk_dots(r, z, r0), world)
    vl = v[r0:r1].copy()
    for k in range(1, max_iters + 1):
        p = gather_rows(p_l, n, world)
        Hp = rowdot(Hl, p)
        pHp = gather_sum(chunk_dots(p_l, Hp, r0), world)
        alpha = rz / pHp
        vl = vl + alpha * p_l
        v = gather_rows(vl, n, world)
        r = bl - rowdot(Hl, v)
        rel = np.sqrt(gather_sum(chunk_dots(r, r, r0), world)) / bnorm
        hist.append(rel)
        if rel <= tol:
            break
        z = r
        rzn = gather_sum(chunk_dots(r, z, r0), world)
        p_l = z + (rzn / rz) * p_l
        rz = rzn
    return v, hist


def sharded_sgd(H, b, rank, world, seed=11, batch=64, lr=0.002, momentum=0.9, iters=60):
    """Row-sharded SGD (solvers.cu sgd_solve_batched over a sharded context): every rank
    draws the same minibatches from the same stream (here numpy, standing in for the
    reference Rng), computes H[row].v - b[row] for the batch rows it owns, updates its own
    velocity/solution rows, all-gathers v, and takes residual norms from chunk partials."""
    n = b.size
    r0, r1 = shard_range(n, world, rank)
    Hl, bl = H[r0:r1], b[r0:r1]
    rng = np.random.default_rng(seed)
    idx = np.arange(n)
    v = np.zeros(n)
    vel_l = np.zeros(r1 - r0)
    bnorm = np.sqrt(gather_sum(chunk_dots(bl, bl, r0), world))
    scale = n / batch
    hist = []
    for _ in range(iters):
        for i in range(batch):  # persistent partial Fisher-Yates
            j = i + int(rng.integers(0, n - i))
            idx[i], idx[j] = idx[j], idx[i]
        rows = idx[:batch].copy()
        vel_l *= momentum
        for row in rows:
            if r0 <= row < r1:
                vel_l[row - r0] += scale * (np.dot(H[row], v) - b[row])
        vl = v[r0:r1] - lr * vel_l
        v = gather_rows(vl, n, world)
        r = bl - rowdot(Hl, v)
        hist.append(np.sqrt(gather_sum(chunk_dots(r, r, r0), world)) / bnorm)
    return v, hist


def sharded_ap(H, b, rank, world, bs=200, iters=40):
    """Row-sharded greedy AP (solvers.cu ap_solve_batched over a sharded context): the
    residual rows a rank owns are updated locally and the full residual is all-gathered
    before each block choice and block solve, so every rank picks the same block and
    applies the same delta to its replicated v."""
    n = b.size
    r0, r1 = shard_range(n, world, rank)
    Hl, bl = H[r0:r1], b[r0:r1]
    nblk = (n + bs - 1) // bs
    chol = [np.linalg.cholesky(H[k * bs:(k + 1) * bs, k * bs:(k + 1) * bs]) for k in range(nblk)]
    v = np.zeros(n)
    bnorm = np.sqrt(gather_sum(chunk_dots(bl, bl, r0), world))
    r_l = bl - rowdot(Hl, v)
    hist = []
    for k in range(1, iters + 1):
        r = gather_rows(r_l, n, world)
        norms = [np.linalg.norm(r[j * bs:(j + 1) * bs]) for j in range(nblk)]
        best = int(np.argmax(norms))  # first maximum
        L = chol[best]
        blk = slice(best * bs, min(n, (best + 1) * bs))
        delta = np.linalg.solve(L.T, np.linalg.solve(L, r[blk]))
        v[blk] += delta
        r_l = r_l - rowdot(Hl[:, blk], delta)
        if k % nblk == 0:
            r_l = bl - rowdot(Hl, v)
        hist.append(np.sqrt(gather_sum(chunk_dots(r_l, r_l, r0), world)) / bnorm)
    return v, hist


def system(n=1300):
    rng = np.random.default_rng(0)
    X = rng.random((n, 3))
    d2 = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    H = np.exp(-0.5 * d2 / 0.3 ** 2) + 0.5 * np.eye(n)
    return H, rng.standard_normal(n)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, b = system()
    v, hist = sharded_cg(H, b, rank, world)
    vs, hs = sharded_sgd(H, b, rank, world)
    va, ha = sharded_ap(H, b, rank, world)
    if rank == 0:
        q.put((v, hist, vs, hs, va, ha))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_solvers_bitwise_equal_single_process(world):
    H, b = system()
    v1, h1 = sharded_cg(H, b, 0, 1)
    vs1, hs1 = sharded_sgd(H, b, 0, 1)
    va1, ha1 = sharded_ap(H, b, 0, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    v2, h2, vs2, hs2, va2, ha2 = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert h1 == h2                      # identical residual histories, bit for bit
    assert np.array_equal(v1, v2)
    assert hs1 == hs2 and np.array_equal(vs1, vs2)  # sharded SGD likewise
    assert hs1[-1] < hs1[0]
    assert ha1 == ha2 and np.array_equal(va1, va2)  # and sharded AP
    assert ha1[-1] < ha1[0]


def test_shard_range_matches_library(W):
    for n in (1, 513, 1300, 101000):
        for world in (1, 2, 3, 8):
            for r in range(world):
                assert W.shard_range(n, world, r) == shard_range(n, world, r)

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
    nch = (n + CHUNK - 1) // CHUNK
    c0, c1 = nch * rank // world, nch * (rank + 1) // world
    return min(c0 * CHUNK, n), min(c1 * CHUNK, n)


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
    if rank == 0:
        q.put((v, hist))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_cg_bitwise_equals_single_process(world):
    H, b = system()
    v1, h1 = sharded_cg(H, b, 0, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    v2, h2 = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert h1 == h2                      # identical residual histories, bit for bit
    assert np.array_equal(v1, v2)


def test_shard_range_matches_library(W):
    for n in (1, 513, 1300, 101000):
        for world in (1, 2, 3, 8):
            for r in range(world):
                assert W.shard_range(n, world, r) == shard_range(n, world, r)

#!/usr/bin/env python
"""Benchmark of the warm-started GP kernel-matvec path (BASELINE.json north_star).

Workload (BASELINE.json configs[2], "C3"): N = 100,000 + 1,000 appended rows,
d = 16, Matern-3/2 (l = 0.8, s_f = 1, sigma_n^2 = 1e-3), X ~ N(0, I), s = 64 RHS.
A step is one fused kernel-matvec (K(X,X) + sigma_n^2 I) V over all N x N pairs and
all 64 right-hand sides.

  value      : kernel-matvec TFLOP/s, algorithmic flops N_r N_c (2d + 2s) per step,
               device-timed with CUDA events, inputs resident in HBM, L2 flushed
               (256 MiB memset) before every step outside the timed events.
  e2e        : the same metric through the public API (wgp_kmatvec via
               warmgp.KernelOperator.kmatvec) with pinned HOST fp64 column-major V
               in and Y out, host<->device copies inside the timed region.
  roofline   : the dominant kernel against the measured peak (MEASURED_PEAKS.json).
  cpu_baseline: the oracle's matrix-free OpenMP restatement of the reference on the
               host cores, on a bounded row sample of the same workload.
  cg         : warm vs cold CG time-to-tolerance (tol 1e-4) on the same system.

``--impl reference`` times the reference's algorithm (CPU oracle port, all host
threads) on the same metric/config and prints one JSON line with impl=reference.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N0, N_APPEND, DIM, S = 100_000, 1_000, 16, 64
LS, SF, NOISE_VAR = 0.8, 1.0, 1e-3
METRIC = "kernel-matvec TFLOP/s (C3: N=101k, d=16, Matern-3/2, s=64)"


def flops_per_matvec(n_rows, n_cols, d=DIM, s=S):
    return float(n_rows) * float(n_cols) * (2 * d + 2 * s)


def make_inputs(seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((N0 + N_APPEND, DIM))
    return X


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_config(n, world):
    """The workload dict of BOTH arms (same metric, same config)."""
    return {"workload": "C3 kernel-matvec (BASELINE configs[2])", "n": n, "d": DIM, "s": S,
            "kernel": "matern32", "lengthscale": LS, "noise_var": NOISE_VAR, "world": world,
            "l2": "flushed (256 MiB memset) before each step"}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


class NvmlClockSampler(ClockSampler):
    """The same samples read in-process through NVML (nvidia-ml-py): no nvidia-smi process
    per sample."""

    def _run(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.device)
        except Exception:
            return
        bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                ("sw_power_cap", 0x4)]
        while not self._stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
                pw = N.nvmlDeviceGetPowerUsage(h) / 1000.0
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx), str(pw)] + ["Active" if r & b else "Not Active" for _, b in bits])
            except Exception:
                pass
            self._stop.wait(0.2)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# --------------------------------------------------------------------------- CPU legs
def cpu_matvec_sample(X, n_rows, nthreads, seed=1):
    """Oracle matrix-free matvec (the reference's per-entry formula) on a row sample."""
    from oracle import oracle as O
    O.build()
    h = O.KernelHyperparams(LS, SF, NOISE_VAR ** 0.5, O.MATERN32)
    V = np.random.default_rng(seed).standard_normal((X.shape[0], S))
    XF = np.asfortranarray(X)
    VF = np.asfortranarray(V)
    t0 = time.perf_counter()
    O.kmatvec(XF, h, VF, rows=(0, n_rows), nthreads=nthreads)
    dt = time.perf_counter() - t0
    return flops_per_matvec(n_rows, X.shape[0]) / dt / 1e12, dt


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    X = make_inputs()
    n = X.shape[0]
    nthreads = os.cpu_count() or 1
    rows = args.ref_rows
    for _ in range(max(args.warmup, 0) and 1):
        cpu_matvec_sample(X, max(rows // 8, 8), nthreads)
    vals = []
    t_all = time.perf_counter()
    for k in range(args.steps):
        v, _ = cpu_matvec_sample(X, rows, nthreads, seed=k + 2)
        vals.append(v)
    wall = time.perf_counter() - t_all
    value = float(np.mean(vals))
    ms = wall / max(args.steps, 1) * 1e3  # one step = one bounded row sample (executed)
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True,
        "ms_full_matvec_extrapolated": flops_per_matvec(n, n) / (value * 1e12) * 1e3, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded X ~ N(0,I))",
        "config": bench_config(n, args.gpus),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": nthreads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{rows} of {n} rows x {n} cols x {S} RHS per step, extrapolated "
                                   f"per-flop to the full matvec (oracle/warmgp_oracle.c "
                                   f"wgo_kmatvec_rows, OpenMP); {args.steps} steps took {wall:.1f} s"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- CG warm/cold
def cg_time_to_tolerance(W, ctx, X, prec, hyp, tol=1e-4, seed=0, local=0):
    """BASELINE configs[2]: solve the N=100k system, append 1000 rows, then warm-started
    ([u; 0], Initialization::warm) vs cold CG to tol on N=101k.  RHS = y + 63 pathwise
    prior samples: 64 Matern RFF priors (F=2048, sample_prior's Student-t spectral draws)
    evaluated on the device plus sigma_n N(0,1) noise (build_sample_rhs).  Times are the
    public solve_many call (host buffers in/out, preconditioner build included)."""
    import numpy as np

    n = X.shape[0]
    priors = [W.sample_prior(hyp, DIM, 2048, W.derive_seed(seed, 100 + c)) for c in range(S)]
    op = W.KernelOperator(hyp, X[:N0], precision=prec, ctx=ctx)
    full = W.KernelOperator(hyp, X, precision=W.F64, ctx=ctx)  # RFF evaluation host (rows only)
    B = W.rff_eval(full, priors)
    del full
    B += hyp.noise_scale * W.normal_fill(W.derive_seed(seed, 3), n * S).reshape(n, S, order="F")
    B = np.asfortranarray(B)
    cfg = W.SolverConfig(tolerance=tol, max_iters=1000, precond_rank=100, precond_shift=hyp.noise_scale ** 2)

    def run(o, rhs, inits):
        if ctx.world > 1:  # sharded: every rank runs the solve; the time is the max over ranks
            import torch
            import torch.distributed as dist
            dist.barrier()
        t0 = time.perf_counter()
        res = W.solve_many(o, rhs, inits, cfg)
        dt = time.perf_counter() - t0
        if ctx.world > 1:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        its = [r.iterations for r in res]
        return res, {"seconds": dt, "iters_max": max(its), "iters_mean": float(np.mean(its)),
                     "converged": int(sum(r.converged for r in res)),
                     "final_rel_residual_max": float(max(r.residual_history[-1] for r in res))}

    prev, prev_stats = run(op, np.asfortranarray(B[:N0]), [W.Initialization.cold()] * S)
    op.append_rows(X[N0:])  # device-resident growth (K8)
    # cold and warm alternately, REPS times each; the solves are deterministic (same
    # iterations, same results), so repeats differ only by host effects and the GPU clock
    # state after the sustained matvec loop.  Reported: the median, every sample, the
    # first call of each, and the SM clocks sampled during the leg.
    reps = 5
    ws, cs = [], []
    with ClockSampler(local) as clk:
        for _ in range(reps):
            _, c = run(op, B, [W.Initialization.cold()] * S)
            _, w = run(op, B, [W.Initialization.warm(r.v) for r in prev])
            cs.append(c)
            ws.append(w)

    def agg(rs):
        out = dict(rs[0])
        secs = [r["seconds"] for r in rs]
        out["seconds"] = float(np.median(secs))
        out["seconds_all"] = secs
        out["seconds_first_call"] = secs[0]
        out["seconds_min"] = float(min(secs))
        return out

    cold, warm = agg(cs), agg(ws)
    return {"n_prev": N0, "n": n, "s": S, "tol": tol, "precond_rank": 100, "reps": reps,
            "statistic": "median of the alternating repetitions (all samples listed)",
            "prev_solve_n100k": prev_stats, "warm": warm, "cold": cold,
            "clocks_during_cg": clk.summary(),
            "warm_over_cold_time": warm["seconds"] / cold["seconds"],
            "warm_over_cold_iters": warm["iters_mean"] / max(cold["iters_mean"], 1e-9)}


def vector_kernels_gbs(W, ctx, n, stream, flush, peaks, reps=20):
    """North-star item (2): the fused solver vector kernels of one CG iteration
    (solvers.cpp:163-180) on [n][S] fp64 arrays at the C3 shape, through the C-ABI device
    entry points, timed with CUDA events on the launching stream, L2 flushed before each
    launch by READING a 256 MiB buffer (a memset flush leaves 126 MB of dirty lines that the
    timed kernel would then have to write back).  Algorithmic bytes: axpy/xpby read two arrays and write one (24 B per element),
    a dot reads two (16 B per element).

    Back-to-back figure (the one compared with the HBM peak): NSETS launches over distinct
    buffer sets bracketed by ONE event pair after one flush -- each launch's inputs are not in
    L2 (the previous launch's 103-155 MB displaced everything else from the 126 MB L2), and
    the ~2-5 us launch/event overhead that a single event-timed ~20 us launch carries is
    amortised."""
    import torch

    dt = torch.float64
    g = torch.Generator(device="cuda").manual_seed(5)
    NSETS = 6
    sets = [(torch.randn(n, S, device="cuda", dtype=dt, generator=g),
             torch.randn(n, S, device="cuda", dtype=dt, generator=g)) for _ in range(NSETS)]
    A, B = sets[0]
    coef = torch.rand(S, device="cuda", dtype=dt, generator=g) + 0.5
    act = torch.ones(S, device="cuda", dtype=torch.int32)
    out = torch.empty(S, device="cuda", dtype=dt)
    work = torch.empty(((n + 511) // 512) * S, device="cuda", dtype=dt)
    sp = stream.cuda_stream
    rd = flush.view(torch.float64)
    sink = torch.empty((), device="cuda", dtype=dt)
    ops = {
        "axpy_cols (v += alpha p)": (lambda A=A, B=B: ctx.axpy_cols_dev(A.data_ptr(), B.data_ptr(), coef.data_ptr(), n, S, sp), 24),
        "xpby_cols (p = z + beta p)": (lambda A=A, B=B: ctx.xpby_cols_dev(A.data_ptr(), B.data_ptr(), coef.data_ptr(),
                                                                          act.data_ptr(), n, S, sp), 24),
        "coldots (p.Hp, r.z, |r|^2)": (lambda A=A, B=B: ctx.coldots_dev(A.data_ptr(), B.data_ptr(), n, S, out.data_ptr(),
                                                                        work.data_ptr(), sp), 16),
    }
    res = {}
    for name, (fn, bpe) in ops.items():
        for _ in range(3):
            fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in ev:
            torch.sum(rd, dim=0, out=sink)  # read-only L2 flush
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
        W.kernel_timer_enable(True)  # second pass: the tagged kernel's own events
        for _ in range(reps):
            torch.sum(rd, dim=0, out=sink)
            fn()
        torch.cuda.synchronize()
        k_ms, k_n = W.kernel_timer_read("coldots")
        W.kernel_timer_enable(False)
        bb = []
        for _ in range(max(3, reps // 4)):
            torch.sum(rd, dim=0, out=sink)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for A_, B_ in sets:
                fn(A_, B_)
            b.record(stream)
            torch.cuda.synchronize()
            bb.append(a.elapsed_time(b) / NSETS)
        bms = float(np.median(bb))
        bgbs = n * S * bpe / (bms * 1e-3) / 1e9
        gbs = n * S * bpe / (ms * 1e-3) / 1e9
        res[name] = {"us": bms * 1e3, "GB/s": bgbs, "frac_hbm": bgbs / peaks["hbm_gbs"],
                     "bytes": n * S * bpe,
                     "timing": f"{NSETS} back-to-back launches over distinct buffer sets per event pair, median of {len(bb)}",
                     "single_launch": {"us": ms * 1e3, "GB/s": gbs, "frac_hbm": gbs / peaks["hbm_gbs"],
                                       "timing": "one launch per event pair (includes launch/event overhead)"}}
        if k_n:  # the HBM-bound kernel alone (the C-ABI call adds the ordered chunk sum, which
            # the solver fuses into its scalar-step kernels)
            kus = k_ms / k_n * 1e3
            res[name]["kernel_only"] = {"us": kus, "GB/s": n * S * bpe / (kus * 1e-6) / 1e9,
                                        "frac_hbm": n * S * bpe / (kus * 1e-6) / 1e9 / peaks["hbm_gbs"]}
    res["shape"] = f"[{n}][{S}] fp64, L2 flushed (256 MiB read) per launch, median of {reps}"
    res["peak_hbm_gbs"] = peaks["hbm_gbs"]
    return res


# --------------------------------------------------------------------------- other hot kernels
def rff_throughput(W, ctx, X, hyp):
    """North-star item (4), RFF prior generation (eval_prior, sampling.cpp:37-46): the
    phase GEMM (d FMA per feature) + cos + amplitude sum per (point, feature, prior).
    fp64 at the C3 right-hand-side shape (101k rows x F=2048 x 64 priors) and the fast fp32
    path at the C5 candidate shape (100k points x F=2000 x 128 priors, d=6), kernel time by
    CUDA events on the launch stream (wgp_kernel_timer, tags rff_eval / rff_eval32)."""
    out = {}
    cases = (("rff_eval (fp64, C3 RHS)", X, S, 2048, DIM, False, hyp),
             ("rff_eval_fast (fp32, C5 candidates)", np.random.default_rng(3).random((100_000, 6)), 128, 2000, 6,
              True, W.KernelHyperparams(0.3, 1.0, 1e-3, W.MATERN32)))
    for name, Xs, nprior, F, d, fast, h in cases:
        op = W.KernelOperator(h, Xs[:1024], precision=W.F64, ctx=ctx)
        priors = [W.sample_prior(h, d, F, W.derive_seed(9, c)) for c in range(nprior)]
        W.rff_eval(op, priors[:2], Xs[:2048], fast=fast)  # warm-up
        W.kernel_timer_enable(True)
        W.rff_eval(op, priors, Xs, fast=fast)
        ms, launches = W.kernel_timer_read("rff_eval32" if fast else "rff_eval")
        W.kernel_timer_enable(False)
        m = Xs.shape[0]
        feats = float(m) * F * nprior
        out[name] = {"kernel_ms": ms, "launches": launches, "points": m, "features": F, "priors": nprior,
                     "dim": d, "cos_per_s": feats / (ms * 1e-3),
                     "algorithmic_flops": feats * (2 * d + 2), "TFLOP/s": feats * (2 * d + 2) / (ms * 1e-3) / 1e12,
                     "note": "flops per (point, feature): 2d (phase) + 2 (amplitude FMA); the cos not counted"}
        del op
    return out


def sgd_ap_kernels(W, ctx):
    """North-star item (3) at the C2 shape (N=20k, d=8 RBF, s=17): SGD minibatch rows
    (krows: B=512 rows x N pairs per column per iteration) and AP block columns (kcols: N x
    bs=500 pairs per column per iteration), fp64, kernel time per launch by CUDA events."""
    from paper_2511_16340_b200 import configs as Cfg
    n, s = 20_000, 17
    hyp = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
    X = Cfg.uniform_rows_fast(W.derive_seed(0, 1), n, 8)
    B = np.asfortranarray(np.random.default_rng(4).standard_normal((n, s)))
    out = {}
    for prec, pname in ((W.F64, "f64"), (W.F32_3XTF32, "f32")):
        op = W.KernelOperator(hyp, X, precision=prec, ctx=ctx)
        for name, tag, kw, pairs in (("sgd", "krows", dict(method=W.SGD, batch_size=512, learning_rate=1e-3), 512 * n),
                                     ("ap", "kcols", dict(method=W.AP, block_size=500), n * 500)):
            cfg = W.SolverConfig(tolerance=1e-12, max_iters=50, **kw)
            W.solve_many(op, B, [W.Initialization.cold()] * s, cfg.copy(max_iters=2))
            W.kernel_timer_enable(True)
            t0 = time.perf_counter()
            W.solve_many(op, B, [W.Initialization.cold()] * s, cfg)
            wall = time.perf_counter() - t0
            ms, launches = W.kernel_timer_read(tag)
            res_ms, res_l = W.kernel_timer_read("kmatvec_tc" if prec != W.F64 else "kmatvec_f64")
            W.kernel_timer_enable(False)
            per = ms / max(launches, 1)
            out[f"{name}_{pname}"] = {
                "kernel": tag, "us_per_launch": per * 1e3, "launches": launches,
                "pairs_per_launch": pairs * s, "Gpairs_per_s": pairs * s / (per * 1e-3) / 1e9,
                "iteration_ms": wall * 1e3 / cfg.max_iters,
                "residual_matvec_ms_per_launch": res_ms / max(res_l, 1),
                "note": "per iteration the reference also recomputes the full true residual (one "
                        "N x N matvec, solvers.cpp:231/:298 refresh) -- listed separately"}
        del op
    out["shape"] = "C2: N=20k, d=8 RBF, s=17; SGD B=512, AP bs=500 (greedy), 50 iterations"
    return out


def c4_sharded_matvec(W, ctx, world, rank, steps=3):
    """C4 (BASELINE configs[3]) operator: N=500k, d=8 RBF, s=32, rows sharded over the ranks
    (all-gather of V + local row slice), device time max over ranks -- the N>=500k scaling
    leg of the north star.  Returns TFLOP/s over all ranks."""
    import torch
    n, d, s = 500_000, 8, 32
    hyp = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
    X = np.random.default_rng(11).random((n, d))
    op = W.KernelOperator(hyp, X, precision=W.F32_3XTF32, ctx=ctx)
    r0, r1 = W.shard_range(n, world, rank)
    V = torch.randn(W.shard_padded_rows(n, world), s, device="cuda", dtype=torch.float64)
    Y = torch.empty(max(r1 - r0, 1), s, device="cuda", dtype=torch.float64)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream

    def step():  # all-gather of the V slots overlapped with the local diagonal block
        op.kmatvec_sharded_dev(V.data_ptr(), Y.data_ptr(), s, sp)

    step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(steps):
        step()
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    flops = float(n) * n * (2 * d + 2 * s)
    return {"n": n, "d": d, "s": s, "kernel": "rbf", "world": world, "ms_per_matvec": ms,
            "TFLOP/s": flops / (ms * 1e-3) / 1e12, "steps": steps,
            "rows_per_rank": r1 - r0,
            "note": "wgp_kmatvec_sharded_dev: all-gather of the V slots (world > 1) overlapped with "
                    "the local diagonal block; device time, max over ranks"}


# --------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2511_16340_b200 import warmgp as W

    prec = {"3xtf32": W.F32_3XTF32, "tf32": W.TF32, "f32simt": W.F32_SIMT, "f64": W.F64}[args.precision]
    if world > 1:
        uid = W.DeviceContext.nccl_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ctx = W.DeviceContext(local, rank, world, obj[0])
    else:
        ctx = W.DeviceContext(local)
    X = make_inputs()
    n = X.shape[0]
    hyp = W.KernelHyperparams(LS, SF, NOISE_VAR ** 0.5, W.MATERN32)
    op = W.KernelOperator(hyp, X[:N0], precision=prec, ctx=ctx)
    op.append_rows(X[N0:])  # the +1000-row growth step (K8)
    assert op.n == n
    r0, r1 = W.shard_range(n, world, rank)
    dt = torch.float64  # device API: fp64 solver vectors for every precision
    gen = torch.Generator(device="cuda").manual_seed(1234)
    V = torch.randn(W.shard_padded_rows(n, world), S, device="cuda", dtype=dt, generator=gen)
    Y = torch.empty(r1 - r0, S, device="cuda", dtype=dt)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()  # a real (non-legacy) stream: our launches and the events share it
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream

    def step():
        if world > 1:  # sharded: all-gather of the V row slots overlapped with the local block
            op.kmatvec_sharded_dev(V.data_ptr(), Y.data_ptr(), S, sp)
        else:
            op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), S, sp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    W.kernel_timer_enable(True)  # CUDA events around the TC kernel launches only
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()  # L2 flush outside the timed events
            starts[k].record(stream)
            step()
            ends[k].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_step = float(np.mean(ms))
    k_ms, k_launches = W.kernel_timer_read()
    W.kernel_timer_enable(False)
    # the tensor-core kernel's time per step (one launch at world 1; the diagonal block and the
    # remote column ranges at world > 1)
    kernel_ms = k_ms / max(1, args.steps)
    t = torch.tensor([ms_step], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    total_flops = flops_per_matvec(n, n)
    value = total_flops / (ms_step * 1e-3) / 1e12

    # e2e through the public API with pinned host buffers (rank 0, unsharded)
    e2e = None
    if world == 1:
        Vh = torch.randn(S, n, dtype=torch.float64, generator=torch.Generator().manual_seed(7)).pin_memory()
        Yh = torch.empty(S, n, dtype=torch.float64).pin_memory()
        Vn, Yn = Vh.numpy().T, Yh.numpy().T  # Fortran-order n x s views
        for _ in range(max(1, args.warmup // 2)):
            op.kmatvec(Vn, out=Yn)
        e2e_ms = []
        for _ in range(max(1, min(args.steps, 20))):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            op.kmatvec(Vn, out=Yn)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_ms_step = float(np.mean(e2e_ms))
        e2e = {"value": total_flops / (e2e_ms_step * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": n * S * 8, "d2h_bytes_per_step": n * S * 8,
               "ms_per_step": e2e_ms_step}
    else:
        # sharded: each rank uploads its V row slice from pinned host memory, the exchange
        # step all-gathers V, the local row slice of H V is computed and read back; the
        # step time is the max over ranks (wall clock around device-synchronised steps)
        Vh = torch.randn(r1 - r0, S, dtype=torch.float64,
                         generator=torch.Generator().manual_seed(7 + rank)).pin_memory()
        Yh = torch.empty(r1 - r0, S, dtype=torch.float64).pin_memory()

        def e2e_step():
            V[r0:r1].copy_(Vh, non_blocking=True)
            step()
            Yh.copy_(Y, non_blocking=True)
            torch.cuda.synchronize()

        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        e2e_ms = []
        for _ in range(max(1, min(args.steps, 20))):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            e2e_step()
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        tm = torch.tensor([float(np.mean(e2e_ms))], device="cuda", dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        e2e_ms_step = float(tm.item())
        e2e = {"value": total_flops / (e2e_ms_step * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": n * S * 8, "d2h_bytes_per_step": n * S * 8,
               "ms_per_step": e2e_ms_step, "note": "all ranks' row slices (bytes summed over ranks)"}

    peaks, peak_kind = measured_peaks()
    # tensor-core roofline.  The contraction is fp32-class (north_star "fp32/tf32"): its
    # tensor format is TF32, dense peak = bf16 dense / 2 on Blackwell (measured bf16 GEMM).
    # The MMAs the kernel issues are kind::f16 three-term hi/lo splits (fp32 accumulate),
    # so the fraction against the f16 dense peak of those instructions is listed as well,
    # and the composite (SFU) bound that actually limits the Matern map.
    # The timed region is 100 back-to-back steps that hold the board at its power cap, i.e. a
    # kernel timed inside a long sustained run: the roofline denominator is the SUSTAINED
    # measured figure (MEASURED_PEAKS.json bf16_tflops_sustained, matmuls back to back for
    # 4 s), the burst one listed alongside.
    peak_tf32_burst = peaks["bf16_tflops"] / 2.0
    sustained = peaks.get("bf16_tflops_sustained")
    peak_tf32 = sustained / 2.0 if sustained else peak_tf32_burst
    peak_f16 = sustained if sustained else peaks["bf16_tflops"]
    sm_hz = peaks.get("sm_max_mhz", 1965.0) * 1e6
    pairs = float(n) * float(n)
    # Matern-3/2: sqrt + exp2 per pair, one exp2 in eight on the FMA pipe (kmatvec_tc.cu
    # WGP_EXP_POLY = 1 of 8 pairs): 1.875 MUFU ops per pair on the SFU
    mufu_per_pair = 2.0 - 1.0 / 8.0
    t_mufu = pairs * mufu_per_pair / (16.0 * 148 * sm_hz)  # 16 MUFU ops/clk/SM
    t_mufu2 = pairs * 2.0 / (16.0 * 148 * sm_hz)
    flops_launch = total_flops / world
    achieved = flops_launch / (kernel_ms * 1e-3) / 1e12 if kernel_ms > 0 else None
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak_tf32, "unit": "TFLOP/s",
            "frac": achieved / peak_tf32 if achieved else None,
            # dram_bytes_read + dram_bytes_write per launch of the TC kernel, from the committed
            # ncu --set full capture of this workload (profiles/r02h_kmatvec_tc_metrics.json):
            # X/XA/XB and the V tiles stay L2-resident, HBM sees little more than V/Y once.
            "traffic": TRAFFIC_BYTES,
            "peak_source": (f"{peak_kind} bf16_tflops_sustained/2 (TF32 dense, sustained: the timed loop "
                            "runs at the board power cap) from MEASURED_PEAKS.json" if sustained else
                            f"{peak_kind} bf16_tflops/2 (TF32 dense) from MEASURED_PEAKS.json"),
            "frac_vs_burst_tf32": achieved / peak_tf32_burst if achieved else None,
            "burst_tf32_peak": peak_tf32_burst,
            "frac_vs_f16_dense": achieved / peak_f16 if achieved else None,
            "f16_dense_peak": peak_f16,
            "mma_kind": "kind::f16, 3-term hi/lo splits of K and V (and of x for the distance "
                        "GEMM), fp32 accumulation in TMEM",
            "kernel": "tc::kmatvec_tc_kernel (CUDA events around its launches, "
                      f"{k_launches} launches over {args.steps} steps, {kernel_ms:.3f} ms per step; "
                      f"{100 * kernel_ms / ms_step:.1f}% of the step)",
            "algorithmic_flops_per_launch": flops_launch,
            "algorithmic_flops_per_pair": 2 * DIM + 2 * S,
            "composite": {"bound": "mufu", "mufu_ops_per_pair": mufu_per_pair,
                          "t_roof_ms": t_mufu * 1e3 / world,
                          "frac": (t_mufu / world) / (kernel_ms * 1e-3) if kernel_ms > 0 else None,
                          "t_roof_ms_2op": t_mufu2 * 1e3 / world,
                          "frac_2op": (t_mufu2 / world) / (kernel_ms * 1e-3) if kernel_ms > 0 else None,
                          "note": "SFU roofline at sm_max_mhz (16 MUFU ops/clk/SM, measured by "
                                  "tools/mufu_microbench.cu): the Matern map's sqrt + exp2 per pair, "
                                  "one exp2 in eight moved to the FMA pipe (1.875 MUFU ops per pair; "
                                  "_2op: the all-MUFU map)"}}

    csum = clk.summary()
    if kernel_ms > 0 and csum.get("sm_mhz"):  # the SFU bound at the clock the loop ran at
        roof["composite"]["frac_at_measured_clock"] = (roof["composite"]["frac"] * sm_hz / 1e6 /
                                                       float(csum["sm_mhz"]))
    vec = rff = sgdap = None
    if world == 1:
        vec = vector_kernels_gbs(W, ctx, n, stream, flush, peaks)
        if not args.no_extra:
            rff = rff_throughput(W, ctx, X, hyp)
            sgdap = sgd_ap_kernels(W, ctx)

    c4 = None
    if not args.no_extra:
        c4 = c4_sharded_matvec(W, ctx, world, rank)

    cg = None
    if not args.no_cg:
        cg = cg_time_to_tolerance(W, ctx, X, prec, hyp, local=local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        nthreads = os.cpu_count() or 1
        v, secs = cpu_matvec_sample(X, args.ref_rows, nthreads)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": nthreads, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"{args.ref_rows} of {n} rows x {n} cols x {S} RHS ({secs:.1f} s), "
                         f"oracle wgo_kmatvec_rows (OpenMP, fp64)"}
        if cg is not None:
            # the CPU CG solve at N=101k is not run (hours); its time is
            # extrapolated from the measured matvec rate: (1 + 2 x iterations) operator
            # applications (the initial residual, then H p and the true residual per
            # iteration, solvers.cpp:150,162,171), preconditioner and vector work excluded.
            t_mv = flops_per_matvec(n, n) / (v * 1e12)
            cpu["cg_extrapolated_s"] = {
                "warm": (1 + 2 * cg["warm"]["iters_max"]) * t_mv,
                "cold": (1 + 2 * cg["cold"]["iters_max"]) * t_mv,
                "basis": "EXTRAPOLATED: (1 + 2 x iters_max) full matvecs at the sampled OpenMP "
                         "oracle rate; preconditioner and vector work excluded"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": {"3xtf32": "f32-class: 3-term fp16 hi/lo splits, fp32 accumulate (kind::f16)",
                      "tf32": "tf32 (single pass)", "f32simt": "f32", "f64": "f64"}[args.precision],
            "data": "synthetic (seeded X ~ N(0,I), V ~ N(0,1))",
            "config": bench_config(n, world),
            "rows_per_rank": r1 - r0,
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "gpu_launches": (5 if world == 1 else 15) * args.steps,  # colmax + colscale_finish + split_v + kmatvec_tc + reduce_splits per launch (world > 1: diagonal block + two remote column ranges)
            "cg_warm_vs_cold": cg,
            "c4_sharded_matvec": c4,
            "vector_kernels": vec,
            "rff_prior_generation": rff,
            "sgd_ap_kernels": sgdap,
            "clocks": clk.summary(), "wall_s": t_wall,
            "step_ms_min": float(np.min(ms)), "step_ms_max": float(np.max(ms)),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# dram bytes (read + write) per launch of tc::kmatvec_tc_kernel on this workload, from the
# committed ncu --set full capture (profiles/r02h_kmatvec_tc_metrics.json: 56.46 MB read + 23.36 MB written)
TRAFFIC_BYTES = 79.82e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # ~0.75 s timed: several clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "tf32", "f32simt", "f64"])
    ap.add_argument("--ref-rows", type=int, default=1000)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cg", action="store_true", help="skip the warm/cold CG time-to-tolerance leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the RFF / SGD-AP / C4 legs")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

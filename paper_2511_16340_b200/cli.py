"""Command-line front end with the reference's `regression-bench` protocol on the device
(reference: proj/tools/warmgp.cpp:115-201, core/src/bench_regression.cpp,
core/src/dataset.cpp, core/src/analysis.cpp:50-87).

    python -m paper_2511_16340_b200.cli regression-bench --data pol.csv --out results \\
        [--device 0] [--precision f64|f32] [the reference's flags]

Same flags and defaults as the reference (RegressionConfig, bench/regression.hpp:14-44),
the same CSV header (`kRegressionCsvHeader`, regression.hpp:63-65) with `%.17g` cells, and
the same `regression_<dataset>.config.txt` sidecar (+ FNV-1a hash).  The protocol per trial
(bench_regression.cpp:129-208): sample_split with the trial seed, median-heuristic
lengthscale, MLL fit on the n1 points, exact solve of the n1 system, growth by n2 rows,
posterior-mean and posterior-sample systems, each configured solver cold and warm.  The
kernel work -- MLL fitting, the exact solve, the RFF sample right-hand side, the growth and
every CG/SGD/AP solve -- runs on the GPU through the C-ABI; dataset parsing, standardization
and the split (host bookkeeping, dataset.cpp) and the warm-start distance report (a dense
diagnostic, analysis.cpp:50-87) run on the host in fp64.
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

import numpy as np

from . import warmgp as W

CSV_HEADER = ("trial,solver,system,init,iters,converged,final_rel_residual,"
              "d_euclid_ratio,d_rkhs_ratio,identity_gap,seed")  # regression.hpp:63-65
METHODS = {"cg": W.CG, "sgd": W.SGD, "ap": W.AP}
NAMES = {v: k for k, v in METHODS.items()}


class ParseError(RuntimeError):
    """types.hpp ParseError: malformed CSV input, naming the offending line."""


def fmt(v: float) -> str:
    """bench_regression.cpp:17-21: %.17g."""
    if isinstance(v, float) and math.isnan(v):
        return "nan"
    return "%.17g" % v


def fnv1a(s: str) -> int:
    """The sidecar hash of bench_regression.cpp:23-30, with the reference's offset constant as
    written there (1469598103934665603, one digit short of the textbook FNV-1a basis), so
    the hashes match the reference's sidecars."""
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & (2**64 - 1)
    return h


# ------------------------------------------------------------------ dataset.cpp restated
def _parse_cell(cell: str):
    c = cell.strip(" \t").rstrip("\r")
    if not c:
        return None
    try:
        return float(c)
    except ValueError:
        return None


def load_csv(path: str, target_column: int, has_header: bool = False):
    """load_csv (dataset.cpp:44-101): numeric CSV, column `target_column` -> y, the rest -> X."""
    try:
        fh = open(path, newline="")
    except OSError:
        raise ParseError(f"cannot open '{path}'")
    rows, arity = [], 0
    with fh:
        for line_no, line in enumerate(fh, start=1):
            line = line.rstrip("\n")
            if line_no == 1 and has_header:
                continue
            if not line or line == "\r":
                continue
            cells = line.split(",")
            if arity == 0:
                arity = len(cells)
                if arity < 2:
                    raise ParseError(f"{path}:{line_no}: need at least two columns")
                if target_column < 0 or target_column >= arity:
                    raise ParseError(f"{path}: target column {target_column} out of range for {arity} columns")
            elif len(cells) != arity:
                raise ParseError(f"{path}:{line_no}: expected {arity} cells, got {len(cells)}")
            vals = []
            for cell in cells:
                v = _parse_cell(cell)
                if v is None:
                    raise ParseError(f"{path}:{line_no}: non-numeric cell '{cell}'")
                vals.append(v)
            rows.append(vals)
    if not rows:
        raise ParseError(f"{path}: no data rows")
    A = np.asarray(rows, dtype=np.float64)
    y = A[:, target_column].copy()
    X = np.delete(A, target_column, axis=1)
    return X, y, os.path.splitext(os.path.basename(path))[0]


def _mean_std(v):
    mean = float(np.mean(v))
    sd = math.sqrt(float(np.sum((v - mean) ** 2)) / v.size)
    if sd <= 1e-12 * (1.0 + abs(mean)):
        sd = 0.0
    return mean, sd


def standardize(X, y):
    """standardize (dataset.cpp:113-140): zero mean, unit population std; constant -> 0."""
    if X.shape[0] < 2:
        raise ValueError("standardize: need at least two rows")
    Xs = np.zeros_like(X)
    for c in range(X.shape[1]):
        m, sd = _mean_std(X[:, c])
        Xs[:, c] = 0.0 if sd == 0.0 else (X[:, c] - m) / sd
    m, sd = _mean_std(y)
    ys = np.zeros_like(y) if sd == 0.0 else (y - m) / sd
    return Xs, ys


def sample_split(X, y, n1: int, n2: int, seed: int):
    """sample_split (dataset.cpp:151-181): partial Fisher-Yates with the reference Rng."""
    if n1 <= 0 or n2 <= 0:
        raise ValueError("sample_split: n1 and n2 must be positive")
    n = X.shape[0]
    if n1 + n2 > n:
        raise ValueError("sample_split: n1 + n2 exceeds dataset size")
    idx = list(range(n))
    rng = W.Rng(seed)
    for i in range(n1 + n2):
        j = i + rng.uniform_index(n - i)
        idx[i], idx[j] = idx[j], idx[i]
    a, b = idx[:n1], idx[n1:n1 + n2]
    return X[a], y[a], X[b], y[b]


# ------------------------------------------------------------------ analysis.cpp:50-87
def warm_start_report(H11, H12, H22, b1, b2):
    """warm_start_report: exact and warm-start distances of the grown system and the
    identity gap (worse of the direct and Schur routes); dense fp64 on the host."""
    n1 = H11.shape[0]
    H = np.block([[H11, H12], [H12.T, H22]])
    b = np.concatenate([b1, b2])
    L = np.linalg.cholesky(H)
    L11 = np.linalg.cholesky(H11)

    def solve(Lf, r):
        return np.linalg.solve(Lf.T, np.linalg.solve(Lf, r))

    v_exact = solve(L, b)
    u1 = solve(L11, b1)
    v_warm = np.zeros_like(b)
    v_warm[:n1] = u1
    d_euclid_cold = float(np.linalg.norm(v_exact))
    d_euclid_warm = float(np.linalg.norm(v_exact - v_warm))
    d_cold_sq = float(b @ v_exact)
    e = v_exact - v_warm
    warm_direct = float(e @ (H @ e))
    warm_schur = warm_direct
    if H22.shape[0] > 0:
        r2 = b2 - H12.T @ u1
        S = H22 - H12.T @ solve(L11, H12)
        warm_schur = float(r2 @ solve(np.linalg.cholesky(S), r2))
    reduction = float(b1 @ u1)
    gap_direct = d_cold_sq - warm_direct - reduction
    gap_schur = d_cold_sq - warm_schur - reduction
    gap = gap_direct if abs(gap_direct) >= abs(gap_schur) else gap_schur
    rk_cold = math.sqrt(max(d_cold_sq, 0.0))
    rk_warm = math.sqrt(max(warm_direct, 0.0))
    return {"euclid_ratio": d_euclid_warm / d_euclid_cold, "rkhs_ratio": rk_warm / rk_cold,
            "identity_gap": gap}


# ------------------------------------------------------------------ bench_regression.cpp
def solver_config_for(a, method, sgd_lr, noise_scale, seed):
    """solver_config_for (bench_regression.cpp:56-76)."""
    max_iters = {W.CG: a.cg_max_iters, W.SGD: a.sgd_max_iters, W.AP: a.ap_max_iters}[method]
    return W.SolverConfig(method=method, tolerance=a.tol, learning_rate=sgd_lr, momentum=a.sgd_momentum,
                          batch_size=a.sgd_batch, sgd_scaling=0, block_size=a.ap_block, precond_rank=a.cg_rank,
                          precond_shift=noise_scale * noise_scale, seed=seed & (2**64 - 1), max_iters=max_iters)


def grid_search_sgd_lr(op, b, a, noise_scale):
    """grid_search_sgd_lr (bench_regression.cpp:80-109): fewest iterations among converged,
    else smallest final residual; diverged rates skipped."""
    best = (a.sgd_lr_grid[0], False, 2**31 - 1, math.inf)
    for lr in a.sgd_lr_grid:
        cfg = solver_config_for(a, W.SGD, lr, noise_scale, 0x9D1D)
        try:
            r = W.solve(op, b, W.Initialization.cold(), cfg)
        except W.DivergenceError:
            continue
        res, iters, conv = r.final_residual(), r.iterations, r.converged
        _, bc, bi, br = best
        better = conv if conv != bc else (iters < bi if conv else res < br)
        if better:
            best = (lr, conv, iters, res)
    return best[0]


def config_text(a, dataset, chosen_lr):
    """config_text (bench_regression.cpp:31-54)."""
    lines = ["command=regression-bench", f"dataset={dataset}", f"data_path={a.data}",
             f"target_column={a.target_col}", f"has_header={1 if a.has_header else 0}",
             f"n1={a.n1}", f"n2={a.n2}", f"trials={a.trials}", f"tolerance={fmt(a.tol)}",
             "solvers=" + ",".join(a.solvers), f"seed={a.seed}", f"mll_steps={a.mll_steps}",
             f"mll_rate={fmt(a.mll_rate)}", f"num_features={a.features}",
             f"sgd_learning_rate={fmt(chosen_lr)}", f"sgd_momentum={fmt(a.sgd_momentum)}",
             f"sgd_batch={a.sgd_batch}", f"ap_block={a.ap_block}", f"cg_rank={a.cg_rank}",
             f"cg_max_iters={a.cg_max_iters}", f"sgd_max_iters={a.sgd_max_iters}",
             f"ap_max_iters={a.ap_max_iters}"]
    return "\n".join(lines) + "\n"


def run_regression_bench(a) -> dict:
    target = a.target_col
    if target < 0:  # negative index: the last column (bench_regression.cpp:210-219)
        target = load_csv(a.data, 0, a.has_header)[0].shape[1]
    X, y, name = load_csv(a.data, target, a.has_header)
    X, y = standardize(X, y)
    if a.n1 <= 0 or a.n2 <= 0 or a.trials <= 0:
        raise ValueError("regression bench: n1, n2 and trials must be positive")
    if a.n1 + a.n2 > X.shape[0]:
        raise ValueError("regression bench: n1 + n2 exceeds dataset size")
    precision = W.F64 if a.precision == "f64" else W.F32_3XTF32
    methods = [METHODS[m] for m in a.solvers]
    sgd_lr = a.sgd_lr
    rows = []

    def flush():
        if not a.out:
            return
        os.makedirs(a.out, exist_ok=True)
        base = os.path.join(a.out, f"regression_{name}")
        with open(base + ".csv", "w") as f:
            f.write(CSV_HEADER + "\n")
            for r in rows:
                f.write(",".join([str(r["trial"]), NAMES[r["solver"]], r["system"], r["init"], str(r["iters"]),
                                  "1" if r["converged"] else "0", fmt(r["final_rel_residual"]),
                                  fmt(r["d_euclid_ratio"]), fmt(r["d_rkhs_ratio"]), fmt(r["identity_gap"]),
                                  str(r["seed"])]) + "\n")
        text = config_text(a, name, sgd_lr)
        with open(base + ".config.txt", "w") as f:
            f.write(text + "config_hash=%x\n" % fnv1a(text))

    try:
        for trial in range(a.trials):
            tseed = W.derive_seed(a.seed, 1000 + trial)
            X1, y1, X2, y2 = sample_split(X, y, a.n1, a.n2, tseed)
            hyp0 = W.KernelHyperparams(W.median_heuristic_lengthscale(X1, tseed), 1.0, 0.1, W.MATERN32)
            hyp = W.optimize_mll(X1, y1, hyp0, a.mll_steps, a.mll_rate)
            Xf = np.vstack([X1, X2])
            op1 = W.KernelOperator(hyp, X1, precision=W.F64)
            # dense blocks for the distance report (host diagnostic, analysis.cpp:50-87)
            H11 = op1.kmatvec(np.eye(a.n1, order="F"))
            H12 = W.cross_kernel(W.KernelOperator(hyp, X2, precision=W.F64), X1)
            H22 = W.KernelOperator(hyp, X2, precision=W.F64).kmatvec(np.eye(a.n2, order="F"))
            op = W.KernelOperator(hyp, X1, precision=precision)
            op.append_rows(X2)  # extend_system: the n1 rows stay resident, n2 appended
            for system in ("mean", "sample"):
                if system == "mean":
                    b1, b2 = y1, y2
                else:
                    prior = W.sample_prior(hyp, Xf.shape[1], a.features, W.derive_seed(tseed, 7))
                    full = W.KernelOperator(hyp, Xf, precision=W.F64)
                    rhs = W.build_sample_rhs(full, prior, hyp.noise_scale, W.derive_seed(tseed, 8))
                    b1, b2 = rhs[:a.n1], rhs[a.n1:]
                u1 = W.exact_solve(op1, b1)
                rep = warm_start_report(H11, H12, H22, b1, b2)
                b = np.concatenate([b1, b2])
                if W.SGD in methods and sgd_lr == 0.0:
                    sgd_lr = grid_search_sgd_lr(op, b, a, hyp.noise_scale)
                for si, m in enumerate(methods):
                    cfg = solver_config_for(a, m, sgd_lr, hyp.noise_scale, W.derive_seed(tseed, 10 + si))
                    for mode in ("cold", "warm"):
                        init = W.Initialization.warm(u1) if mode == "warm" else W.Initialization.cold()
                        row = {"trial": trial, "solver": m, "system": system, "init": mode,
                               "identity_gap": rep["identity_gap"], "seed": tseed,
                               "d_euclid_ratio": rep["euclid_ratio"] if mode == "warm" else 1.0,
                               "d_rkhs_ratio": rep["rkhs_ratio"] if mode == "warm" else 1.0}
                        try:
                            res = W.solve(op, b, init, cfg)
                            row.update(iters=res.iterations, converged=res.converged,
                                       final_rel_residual=res.final_residual())
                        except W.DivergenceError as e:
                            row.update(iters=e.iterations, converged=False, final_rel_residual=float("nan"))
                        rows.append(row)
    finally:
        flush()
    return {"dataset": name, "rows": rows, "chosen_sgd_lr": sgd_lr}


# ------------------------------------------------------------------ thompson.cpp restated
THOMPSON_CSV_HEADER = ("round,init,solver,lengthscale,seed,best_value,mean_residual,"
                       "avg_sample_residual,wall_clock_s")  # bench/thompson.hpp:28-30
BUDGETS = {"small": (5, 120, 30), "large": (25, 600, 150)}  # BoBudget, thompson.hpp:19-27
_PRIMES = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71, 73, 79, 83, 89, 97,
           101, 103, 107, 109, 113, 127, 131, 137, 139, 149, 151]


def short_num(v: float) -> str:
    """std::ostream default formatting (bench_thompson.cpp:22-26)."""
    return "%g" % v


def nth_prime(k: int) -> int:
    """nth_prime (thompson.cpp:69-91)."""
    if k < len(_PRIMES):
        return _PRIMES[k]
    cand, found = _PRIMES[-1], len(_PRIMES) - 1
    while found < k:
        cand += 1
        if all(cand % q for q in range(2, int(cand ** 0.5) + 1)):
            found += 1
    return cand


def radical_inverse(i: int, base: int) -> float:
    inv = 1.0 / base
    f, x = inv, 0.0
    while i > 0:
        x += (i % base) * f
        i //= base
        f *= inv
    return x


def init_design(dim: int, n: int, seed: int) -> np.ndarray:
    """init_design (thompson.cpp:107-124): Halton rows 1..n, shifted mod 1 by a seeded vector."""
    if dim < 1 or n < 1:
        raise ValueError("init_design: dim and n must be positive")
    rng = W.Rng(W.derive_seed(seed, 0xDE5160))
    shift = [rng.uniform() for _ in range(dim)]
    X = np.zeros((n, dim))
    for d in range(dim):
        base = nth_prime(d)
        for i in range(n):
            v = radical_inverse(i + 1, base) + shift[d]
            X[i, d] = v - math.floor(v)
    return X


def propose_candidates(X_obs, y_obs, count, lengthscale, exploration_fraction, temperature_scale, seed):
    """propose_candidates (thompson.cpp:126-183): a uniform share, the rest perturbed copies of
    observed points drawn from softmax(y / T), T = scale * std(y)."""
    n, dim = X_obs.shape
    if n < 1:
        raise ValueError("propose_candidates: no observations")
    if count < 1:
        raise ValueError("propose_candidates: count must be positive")
    n_uniform = min(count, int(math.ceil(exploration_fraction * count)))
    rng = W.Rng(seed)
    cands = np.zeros((count, dim))
    for i in range(n_uniform):
        for d in range(dim):
            cands[i, d] = rng.uniform()
    if n_uniform < count:
        mean = float(np.mean(y_obs))
        sd = math.sqrt(float(np.sum((y_obs - mean) ** 2)) / n)
        temperature = temperature_scale * sd
        if not temperature > 0.0:
            best = int(np.argmax(y_obs))
            cumulative = np.zeros(n)
            cumulative[best:] = 1.0
        else:
            ymax = float(np.max(y_obs))
            cumulative = np.zeros(n)
            total = 0.0
            for i in range(n):
                total += math.exp((y_obs[i] - ymax) / temperature)
                cumulative[i] = total
            cumulative /= total
        perturb_sd = 0.5 * lengthscale
        for i in range(n_uniform, count):
            u = rng.uniform()
            lo, hi = 0, n - 1
            while lo < hi:
                mid = (lo + hi) // 2
                if cumulative[mid] < u:
                    lo = mid + 1
                else:
                    hi = mid
            for d in range(dim):
                cands[i, d] = min(max(X_obs[lo, d] + perturb_sd * rng.normal(), 0.0), 1.0)
    return cands


def run_bo(a, lengthscale: float, init_mode: str, solver: str, seed: int) -> list:
    """run_bo / bo_init / bo_round (thompson.cpp:260-448) with the solves, the posterior
    evaluations at the candidates (select_peaks' argmax) and the Adam peak ascent on the
    device; returns the TrialRecords (round 0 = the initial design)."""
    from . import configs as Cfg

    hyp = W.KernelHyperparams(lengthscale, a.signal_scale, a.noise_scale, W.MATERN32)
    cg_it, sgd_it, ap_it = BUDGETS[a.budget]
    method = METHODS[solver]
    scfg = W.SolverConfig(method=method, tolerance=a.tol, max_iters={W.CG: cg_it, W.SGD: sgd_it, W.AP: ap_it}[method],
                          learning_rate=a.sgd_lr, momentum=a.sgd_momentum, batch_size=a.sgd_batch,
                          block_size=a.ap_block, precond_rank=a.cg_rank, precond_shift=a.noise_scale ** 2)
    # bo_init: objective (make_objective), design, priors, noise draws
    obj_seed = W.derive_seed(seed, 1)
    g = W.sample_prior(hyp, a.dim, 2000, W.derive_seed(obj_seed, 0x0B1EC7))
    obj_rng = W.Rng(W.derive_seed(obj_seed, 0x0B5E7E))
    X0 = init_design(a.dim, a.n_init, W.derive_seed(seed, 2))
    probe = W.KernelOperator(hyp, X0, precision=W.F64)

    def observe(Xn):
        vals = W.rff_eval(probe, [g], Xn)[:, 0]
        return np.array([v + a.noise_scale * obj_rng.normal() for v in vals])

    y0 = observe(X0)
    st = Cfg.growth_state(X0, y0, hyp, a.samples, a.features, seed)
    recs = [{"round": 0, "best_value": float(np.max(y0)), "mean_residual": float("nan"),
             "avg_sample_residual": float("nan"), "wall_clock_s": 0.0}]
    Xobs = X0  # host copy of the observed rows (the operator holds them on the device)
    for _ in range(a.rounds):
        t0 = time.perf_counter()
        rec = st.solve_round(scfg, init_mode == "warm")
        wd = st.weights[:, :1] - st.weights[:, 1:]  # mean - sample_s (pathwise samples)
        peaks = np.zeros((a.samples, a.proposal_rounds, a.dim))
        for rep in range(a.proposal_rounds):
            cands = propose_candidates(Xobs, st.y, a.proposal_count, lengthscale, a.exploration_fraction,
                                       1.0, W.derive_seed(W.derive_seed(seed, 0xA0000 + st.round), rep))
            idx = W.posterior_select(st.op, st.priors, wd, cands, groups=1, fast=False)
            peaks[:, rep, :] = cands[idx[:, 0]]
        pts, _ = W.ascend_peaks(st.op, st.priors, wd, peaks, a.ascent_steps, a.ascent_rate)
        Xn = pts[: a.batch]
        yn = observe(Xn)
        st.add_points(Xn, yn)
        Xobs = np.vstack([Xobs, Xn])
        recs.append({"round": st.round, "best_value": float(np.max(st.y)), "mean_residual": rec["mean_residual"],
                     "avg_sample_residual": rec["avg_sample_residual"],
                     "wall_clock_s": time.perf_counter() - t0})
    return recs


def thompson_config_text(a) -> str:
    """config_text (bench_thompson.cpp:40-72)."""
    cg_it, sgd_it, ap_it = BUDGETS[a.budget]
    lines = ["command=thompson-bench", f"dim={a.dim}", f"n_init={a.n_init}", f"samples={a.samples}",
             f"batch={a.batch}", f"rounds={a.rounds}", f"budget_cg={cg_it}", f"budget_sgd={sgd_it}",
             f"budget_ap={ap_it}", f"tolerance={short_num(a.tol)}", f"signal_scale={short_num(a.signal_scale)}",
             f"noise_scale={short_num(a.noise_scale)}", f"num_features={a.features}",
             f"proposal_count={a.proposal_count}", f"proposal_rounds={a.proposal_rounds}",
             f"ascent_steps={a.ascent_steps}", f"ascent_rate={short_num(a.ascent_rate)}",
             f"exploration_fraction={short_num(a.exploration_fraction)}",
             f"sgd_learning_rate={short_num(a.sgd_lr)}", f"sgd_momentum={short_num(a.sgd_momentum)}",
             f"sgd_batch={a.sgd_batch}", f"ap_block={a.ap_block}", f"cg_rank={a.cg_rank}",
             f"seed_base={a.seed_base}", f"n_seeds={a.seeds}",
             "lengthscales=" + ",".join(short_num(v) for v in a.lengthscales),
             "solvers=" + ",".join(a.solvers), "inits=" + ",".join(a.inits)]
    return "\n".join(lines) + "\n"


def run_thompson_bench(a) -> list:
    """run_thompson_bench (bench_thompson.cpp:76-116): every (lengthscale, seed, init, solver);
    one CSV per (lengthscale, seed, init) with a row per (solver, round)."""
    if a.samples < 1 or a.batch < 1 or a.batch > a.samples or a.n_init < 1 or a.dim < 1:
        raise ValueError("BoConfig: counts must be positive" if a.batch <= a.samples else
                         "BoConfig: batch_size cannot exceed n_samples (one acquisition per posterior sample)")
    runs = []
    if a.out:
        os.makedirs(a.out, exist_ok=True)
        text = thompson_config_text(a)
        with open(os.path.join(a.out, "thompson.config.txt"), "w") as f:
            f.write(text + "config_hash=%x\n" % fnv1a(text))
    for li, ls in enumerate(a.lengthscales):
        for si in range(a.seeds):
            run_seed = W.derive_seed(a.seed_base, (li + 1) * 10000 + si)
            for mode in a.inits:
                file_runs = []
                for solver in a.solvers:
                    run = {"lengthscale": ls, "seed": run_seed, "init": mode, "solver": solver,
                           "records": run_bo(a, ls, mode, solver, run_seed)}
                    runs.append(run)
                    file_runs.append(run)
                if a.out:
                    path = os.path.join(a.out, f"thompson_l{short_num(ls)}_s{si}_{mode}.csv")
                    with open(path, "w") as f:
                        f.write(THOMPSON_CSV_HEADER + "\n")
                        for run in file_runs:
                            for r in run["records"]:
                                f.write(",".join([str(r["round"]), mode, run["solver"], short_num(ls), str(run_seed),
                                                  fmt(r["best_value"]), fmt(r["mean_residual"]),
                                                  fmt(r["avg_sample_residual"]), fmt(r["wall_clock_s"])]) + "\n")
    return runs


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="warmgp-gpu", description="warmgp on the B200: warm-started iterative "
                                 "GP posterior solvers")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("regression-bench", help="Warm versus cold solves on a growing regression dataset")
    # the reference's options and defaults (tools/warmgp.cpp:119-143, bench/regression.hpp:14-44)
    r.add_argument("--data", required=True)
    r.add_argument("--target-col", type=int, default=-1)
    r.add_argument("--has-header", action="store_true")
    r.add_argument("--n1", type=int, default=1000)
    r.add_argument("--n2", type=int, default=100)
    r.add_argument("--trials", type=int, default=10)
    r.add_argument("--tol", type=float, default=0.01)
    r.add_argument("--solvers", type=lambda s: s.split(","), default=["cg", "sgd", "ap"])
    r.add_argument("--out", default="")
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--mll-steps", type=int, default=200)
    r.add_argument("--mll-rate", type=float, default=0.1)
    r.add_argument("--features", type=int, default=2000)
    r.add_argument("--sgd-lr", type=float, default=0.0)
    r.add_argument("--sgd-lr-grid", type=lambda s: [float(v) for v in s.split(",")], default=[0.03, 0.1, 0.3, 1.0])
    r.add_argument("--sgd-momentum", type=float, default=0.9)
    r.add_argument("--sgd-batch", type=int, default=100)
    r.add_argument("--ap-block", type=int, default=100)
    r.add_argument("--cg-rank", type=int, default=100)
    r.add_argument("--cg-max-iters", type=int, default=2000)
    r.add_argument("--sgd-max-iters", type=int, default=30000)
    r.add_argument("--ap-max-iters", type=int, default=5000)
    # device selection (this front end's additions)
    r.add_argument("--device", type=int, default=0)
    r.add_argument("--precision", choices=["f64", "f32"], default="f64",
                   help="operator precision of the solves (f32: the 3-term fp16 tensor-core path)")
    t = sub.add_parser("thompson-bench", help="Budgeted parallel Thompson sampling, warm versus cold")
    # the reference's options and defaults (tools/warmgp.cpp:145-180, thompson.hpp:29-58,
    # bench/thompson.hpp:11-19)
    t.add_argument("--dim", type=int, default=3)
    t.add_argument("--n-init", type=int, default=500)
    t.add_argument("--samples", type=int, default=None)
    t.add_argument("--batch", type=int, default=None)
    t.add_argument("--rounds", type=int, default=10)
    t.add_argument("--budget", choices=["small", "large"], default="small")
    t.add_argument("--lengthscales", type=lambda s: [float(v) for v in s.split(",")], default=[0.1, 0.2, 0.3, 0.4, 0.5])
    t.add_argument("--seeds", type=int, default=2)
    t.add_argument("--seed-base", type=int, default=0)
    t.add_argument("--solvers", type=lambda s: s.split(","), default=["cg", "sgd", "ap"])
    t.add_argument("--inits", type=lambda s: s.split(","), default=["warm", "cold"])
    t.add_argument("--features", type=int, default=2000)
    t.add_argument("--tol", type=float, default=1e-2)
    t.add_argument("--signal-scale", type=float, default=1.0)
    t.add_argument("--noise-scale", type=float, default=1e-3)
    t.add_argument("--proposal-count", type=int, default=250)
    t.add_argument("--proposal-rounds", type=int, default=5)
    t.add_argument("--ascent-steps", type=int, default=30)
    t.add_argument("--ascent-rate", type=float, default=0.05)
    t.add_argument("--exploration-fraction", type=float, default=0.1)
    t.add_argument("--sgd-lr", type=float, default=0.3)
    t.add_argument("--sgd-momentum", type=float, default=0.9)
    t.add_argument("--sgd-batch", type=int, default=100)
    t.add_argument("--ap-block", type=int, default=100)
    t.add_argument("--cg-rank", type=int, default=100)
    t.add_argument("--out", default="")
    t.add_argument("--summary", action="store_true")
    t.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "regression-bench":
            for m in a.solvers:
                if m not in METHODS:
                    raise ValueError(f"unknown solver '{m}'")
            if a.device != 0:  # every operator below is created on the default context
                W._default_ctx = W.DeviceContext(a.device)
            out = run_regression_bench(a)
            msg = f"dataset {out['dataset']}: {len(out['rows'])} rows"
            if a.out:
                msg += f" -> {a.out}/regression_{out['dataset']}.csv"
            print(msg)
            if out["chosen_sgd_lr"] > 0.0:
                print(f"sgd learning rate: {out['chosen_sgd_lr']:g}")
        elif a.cmd == "thompson-bench":
            for m in a.solvers:
                if m not in METHODS:
                    raise ValueError(f"unknown solver '{m}'")
            for m in a.inits:
                if m not in ("warm", "cold"):
                    raise ValueError(f"unknown init mode '{m}'")
            # --samples without --batch: one acquisition per sample (tools/warmgp.cpp:203-205)
            if a.samples is None:
                a.samples = 10
                a.batch = 10 if a.batch is None else a.batch
            elif a.batch is None:
                a.batch = a.samples
            if a.device != 0:
                W._default_ctx = W.DeviceContext(a.device)
            runs = run_thompson_bench(a)
            print(f"{len(runs)} runs" + (f" -> {a.out}" if a.out else ""))
            if a.summary:  # tools/warmgp.cpp:64-83
                best, resid = {}, {}
                for r in runs:
                    key = (r["init"], r["solver"])
                    best.setdefault(key, []).append(r["records"][-1]["best_value"])
                    resid.setdefault(key, []).append(r["records"][-1]["mean_residual"])
                print("final round, mean +- stderr over runs:")
                for key in sorted(best):
                    v = np.asarray(best[key])
                    se = math.sqrt(float(np.sum((v - v.mean()) ** 2)) / (v.size - 1) / v.size) if v.size > 1 else 0.0
                    print(f"  {key[1]} {key[0]}: best {v.mean():g} +- {se:g}, mean residual {np.mean(resid[key]):g}")
    except Exception as e:  # noqa: BLE001  (tools/warmgp.cpp:209-212)
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())

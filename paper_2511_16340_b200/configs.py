"""Drivers for the BASELINE.json configurations over the warmgp API (callers of the path).

The sequential-growth bookkeeping restates bo_round's warm-start half
(thompson.cpp:321-386, 403-422): rows are appended to the device-resident operator,
the right-hand sides are [y | prior_s(X) + noise_s] (thompson.cpp:343-347), warm
initialisations are the previous weights zero-extended (:349-356), per-column SGD
seeds are derive_seed(derive_seed(seed, 0xc0000 + round), col) (:372), divergence
keeps the initial weights with a one-entry history (solve_best_effort :299-317), and
the prior values / noise of new rows are drawn in the reference's order (:415-422,
noise i-major then sample).  The acquisition of configuration 5 evaluates the posterior
samples at 100k uniform candidates, takes each sample's argmax in every candidate group
as Adam starting points and ascends them on the device (select_peaks + ascend_peaks,
thompson.cpp:188-258); the reference's anchored candidate proposal
(propose_candidates, thompson.cpp:160-185) is replaced by uniform candidates.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import warmgp as W


def uniform_rows(seed: int, n: int, d: int) -> np.ndarray:
    """n x d U[0,1) rows in testutil.hpp:9-16 order (reference Rng)."""
    r = W.Rng(seed)
    X = np.empty((n, d))
    for i in range(n):
        for k in range(d):
            X[i, k] = r.uniform()
    return X


def uniform_rows_fast(seed: int, n: int, d: int) -> np.ndarray:
    """Same stream as uniform_rows, vectorised through the oracle-independent splitmix64."""
    z = (np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * np.arange(1, n * d + 1, dtype=np.uint64))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53).reshape(n, d)


@dataclass
class GrowthState:
    """BoState (thompson.hpp:108-123) minus the objective/acquisition parts."""
    op: W.KernelOperator
    hyp: W.KernelHyperparams
    priors: list
    y: np.ndarray                 # n
    prior_values: np.ndarray      # n x S
    noise_draws: np.ndarray       # n x S
    noise_rng: W.Rng
    seed: int = 0
    weights: np.ndarray | None = None   # n_solved x (1 + S)
    n_solved: int = 0
    round: int = 0
    history: list = field(default_factory=list)
    op_fast: W.KernelOperator | None = None  # tensor-core twin of op for candidate evaluation

    @property
    def n_obs(self) -> int:
        return self.op.n

    def rhs(self) -> np.ndarray:
        """[y | prior_values + noise_draws] (thompson.cpp:343-347)."""
        return np.asfortranarray(np.column_stack([self.y, self.prior_values + self.noise_draws]))

    def solve_round(self, cfg: W.SolverConfig, warm: bool) -> dict:
        """Budgeted solves of all columns, warm or cold (thompson.cpp:349-386)."""
        self.round += 1
        B = self.rhs()
        s = B.shape[1]
        use_warm = warm and self.n_solved > 0
        inits = ([W.Initialization.warm(self.weights[:, c]) for c in range(s)] if use_warm
                 else [W.Initialization.cold()] * s)
        c = cfg.copy(seed=W.derive_seed(self.seed, 0xC0000 + self.round))
        t0 = time.perf_counter()
        res, status, dv = W.solve_many(self.op, B, inits, c, return_status=True)
        t_solve = time.perf_counter() - t0
        for col in range(s):  # solve_best_effort (thompson.cpp:299-317)
            if status[col] == W.DIVERGED:
                n1 = self.n_solved if use_warm else 0
                v0 = W.init_weights(inits[col], n1, self.n_obs - n1)
                r = self.op.kmatvec(v0) - B[:, col]
                res[col] = W.SolveResult(v0, int(dv[col]), [float(np.linalg.norm(r) / np.linalg.norm(B[:, col]))], False)
        self.weights = np.column_stack([r.v for r in res])
        self.n_solved = self.n_obs
        rec = {"round": self.round, "n": self.n_obs, "warm": use_warm, "seconds": t_solve,
               "mean_iterations": res[0].iterations, "mean_residual": res[0].final_residual(),
               "max_sample_iterations": max(r.iterations for r in res[1:]) if s > 1 else 0,
               "avg_sample_residual": float(np.mean([r.final_residual() for r in res[1:]])) if s > 1 else 0.0,
               "iterations": [r.iterations for r in res], "converged": int(sum(r.converged for r in res)),
               "diverged": int(sum(status == W.DIVERGED)), "anchors": self.op.last_anchor_count}
        self.history.append(rec)
        return rec

    def add_points(self, Xn: np.ndarray, yn: np.ndarray):
        """Append a batch: observations, prior values at the new rows, noise draws
        (thompson.cpp:403-422)."""
        Xn = np.asarray(Xn, dtype=np.float64)
        m = Xn.shape[0]
        S = len(self.priors)
        pv = W.rff_eval(self.op, self.priors, Xn) if S else np.zeros((m, 0))
        nd = self.noise_rng.normal_fill(m * S, self.hyp.noise_scale).reshape(m, S)  # i-major
        self.op.append_rows(Xn)
        if self.op_fast is not None:
            self.op_fast.append_rows(Xn)
        self.y = np.concatenate([self.y, yn])
        self.prior_values = np.vstack([self.prior_values, pv])
        self.noise_draws = np.vstack([self.noise_draws, nd])


def growth_state(X0, y0, hyp, n_samples, num_features, seed, precision=W.F64, ctx=None,
                 residual=W.RESIDUAL_DIRECT) -> GrowthState:
    """bo_init's sampling half (thompson.cpp:260-293): priors derive_seed(seed, 100 + s),
    prior values at the initial design, noise from Rng(derive_seed(seed, 3)) i-major."""
    op = W.KernelOperator(hyp, X0, precision=precision, ctx=ctx, residual=residual)
    d = X0.shape[1]
    priors = [W.sample_prior(hyp, d, num_features, W.derive_seed(seed, 100 + s)) for s in range(n_samples)]
    pv = W.rff_eval(op, priors) if n_samples else np.zeros((X0.shape[0], 0))
    rng = W.Rng(W.derive_seed(seed, 3))
    nd = rng.normal_fill(X0.shape[0] * n_samples, hyp.noise_scale).reshape(X0.shape[0], n_samples)
    return GrowthState(op, hyp, priors, np.asarray(y0, dtype=np.float64).copy(), pv, nd, rng, seed)


# ----------------------------------------------------------------------------------- C5
@dataclass
class BumpObjective:
    """Configuration 5's objective: sum of 20 seeded Gaussian bumps on [0,1]^D plus
    N(0, 0.01) observation noise (builder-defined; replaces make_objective)."""
    centers: np.ndarray
    widths: np.ndarray
    amps: np.ndarray
    noise_rng: W.Rng
    noise_std: float = 0.1

    @staticmethod
    def make(dim: int, seed: int, n_bumps: int = 20) -> "BumpObjective":
        r = W.Rng(W.derive_seed(seed, 0x0B1EC7))
        c = np.array([[r.uniform() for _ in range(dim)] for _ in range(n_bumps)])
        w = np.array([r.uniform(0.05, 0.2) for _ in range(n_bumps)])
        a = np.array([r.uniform(0.5, 1.5) for _ in range(n_bumps)])
        return BumpObjective(c, w, a, W.Rng(W.derive_seed(seed, 0x0B5E7E)))

    def value(self, X: np.ndarray) -> np.ndarray:
        d2 = ((X[:, None, :] - self.centers[None, :, :]) ** 2).sum(-1)
        return (self.amps[None, :] * np.exp(-0.5 * d2 / self.widths[None, :] ** 2)).sum(-1)

    def observe(self, X: np.ndarray) -> np.ndarray:
        v = self.value(X)
        return v + self.noise_rng.normal_fill(v.size, self.noise_std)


def posterior_at(state: GrowthState, Xc: np.ndarray) -> np.ndarray:
    """eval_posterior (sampling.cpp:66-75) for every sample at once on the device:
    prior_s(X*) + K(X*, X)(w_mean - w_s)  ->  m x S.  With a tensor-core twin operator the
    candidates go through the tcgen05 cross mode and the fp32 RFF kernel (acquisition only
    ranks the values; the solves stay on the fp64 operator)."""
    Wd = state.weights[:, :1] - state.weights[:, 1:]
    if state.op_fast is not None:
        return W.rff_eval(state.op_fast, state.priors, Xc, fast=True) + state.op_fast.cross_matvec(Xc, Wd)
    return W.rff_eval(state.op, state.priors, Xc) + state.op.cross_matvec(Xc, Wd)


def bo_loop(dim=4, n_init=5000, batch=64, rounds=50, n_samples=128, candidates=100_000,
            warm=True, seed=0, cfg: W.SolverConfig | None = None, precision=W.F64, ctx=None,
            fast_candidates: bool = True, peak_groups: int = 5, ascent_steps: int = 30,
            ascent_rate: float = 0.05) -> dict:
    """Configuration 5: BoConfig defaults (Matern-3/2 l=0.3, s_f=1, sigma_n=1e-3, F=2000;
    thompson.hpp:29-58), CG with the small budget (5 iterations, tol 1e-2).  Acquisition as
    select_peaks + ascend_peaks (thompson.cpp:188-258): the candidates are split into
    `peak_groups` contiguous groups [m g / G, m (g+1) / G), each sample's argmax in every group
    (computed on the device, wgp_posterior_select) is a start, and the device Adam
    ascent (ascent_steps / ascent_rate, BoConfig defaults 30 / 0.05) picks the batch point;
    ascent_steps = 0 takes the plain argmax."""
    hyp = W.KernelHyperparams(0.3, 1.0, 1e-3, W.MATERN32)
    cfg = cfg or W.SolverConfig(method=W.CG, tolerance=1e-2, max_iters=5, precond_rank=100,
                                precond_shift=hyp.noise_scale ** 2)
    obj = BumpObjective.make(dim, seed)
    X0 = uniform_rows_fast(W.derive_seed(seed, 2), n_init, dim)
    y0 = obj.observe(X0)
    st = growth_state(X0, y0, hyp, n_samples, 2000, seed, precision, ctx)
    if fast_candidates:
        st.op_fast = W.KernelOperator(hyp, X0, precision=W.F32_3XTF32, ctx=ctx)
    recs = []
    for r in range(rounds):
        rec = st.solve_round(cfg, warm)
        t0 = time.perf_counter()
        Xc = uniform_rows_fast(W.derive_seed(seed, 0xA0000 + st.round), candidates, dim)
        # select_peaks on the device: posterior values of the first `batch` samples at every
        # candidate and their per-group argmax; only batch x groups indices reach the host
        wd = st.weights[:, :1] - st.weights[:, 1:1 + batch]
        sel_op = st.op_fast if st.op_fast is not None else st.op
        groups = peak_groups if ascent_steps > 0 else 1
        idx = W.posterior_select(sel_op, st.priors[:batch], wd, Xc, groups=groups,
                                 fast=st.op_fast is not None)
        if ascent_steps > 0:
            starts = Xc[idx]  # batch x groups x D
            Xn, _ = W.ascend_peaks(st.op, st.priors[:batch], wd, starts, ascent_steps, ascent_rate)
        else:
            Xn = Xc[idx[:, 0]]
        rec["candidate_seconds"] = time.perf_counter() - t0
        yn = obj.observe(Xn)
        st.add_points(Xn, yn)
        rec["best_value"] = float(st.y.max())
        recs.append(rec)
    return {"dim": dim, "warm": warm, "rounds": recs,
            "total_solve_seconds": float(sum(r["seconds"] for r in recs)),
            "total_candidate_seconds": float(sum(r["candidate_seconds"] for r in recs))}


# ----------------------------------------------------------------------------------- C2
def grid_search_sgd_lr(op, b, cfg: W.SolverConfig, grid=(0.03, 0.1, 0.3, 1.0)) -> float:
    """grid_search_sgd_lr (bench_regression.cpp:79-109): cold SGD on a probe system per
    grid rate (seed 0x9d1d); converged-in-fewest wins, else smallest final residual."""
    best_lr, best_conv, best_it, best_res = grid[0], False, 1 << 30, float("inf")
    for lr in grid:
        try:
            r = W.sgd_solve(op, b, W.Initialization.cold(), cfg.copy(learning_rate=lr, seed=0x9D1D))
        except W.DivergenceError:
            continue
        conv, it, res = r.converged, r.iterations, r.final_residual()
        better = (conv if conv != best_conv else (it < best_it if conv else res < best_res))
        if better:
            best_lr, best_conv, best_it, best_res = lr, conv, it, res
    return best_lr



def growth_sweep(method=W.CG, steps=range(21), n0=10_000, step=500, pool=20_000, d=8, n_samples=16,
                 precision=W.F64, tol=1e-4, max_iters=2000, seed=0, lr=None, ctx=None,
                 residual=W.RESIDUAL_DIRECT) -> dict:
    """Configuration 2: RBF (l=0.5, s_f=1, sigma_n^2=1e-2), systems N = n0 + step*t drawn from
    a fixed pool, s = 17 (y + 16 pathwise samples, F=1024), warm (previous step's solution
    zero-extended) vs cold, per solver (AP block 500 greedy, SGD batch 512)."""
    hyp = W.KernelHyperparams(0.5, 1.0, 0.1, W.RBF)
    Xp = uniform_rows_fast(W.derive_seed(seed, 1), pool, d)
    fy = W.sample_prior(hyp, d, 1024, W.derive_seed(seed, 7))
    tmp = W.KernelOperator(hyp, Xp, precision=W.F64, ctx=ctx)
    yp = W.rff_eval(tmp, [fy])[:, 0] + W.normal_fill(W.derive_seed(seed, 8), pool, hyp.noise_scale)
    del tmp
    cfg = W.SolverConfig(method=method, tolerance=tol, max_iters=max_iters, precond_rank=100,
                         precond_shift=hyp.noise_scale ** 2, block_size=500, batch_size=512,
                         learning_rate=lr if lr is not None else 0.3, seed=seed)
    out = {"method": method, "precision": precision, "residual": residual, "steps": []}
    states = {}
    for mode in ("warm", "cold"):
        st = growth_state(Xp[:n0], yp[:n0], hyp, n_samples, 1024, seed, precision, ctx, residual)
        states[mode] = st
    ts = list(steps)
    for t in range(max(ts) + 1):
        n_t = n0 + step * t
        for mode, st in states.items():
            if st.n_obs < n_t:
                st.add_points(Xp[st.n_obs:n_t], yp[st.n_obs:n_t])
            if t in ts:
                rec = st.solve_round(cfg, warm=(mode == "warm"))
                rec["t"] = t
                out["steps"].append({"mode": mode, **rec})
            elif mode == "warm":
                # keep the warm chain: solve every step (only recorded ones are reported)
                st.solve_round(cfg, warm=True)
    return out

"""Probe (not collected): per-tile clock trace of CTA 0 of the tcgen05 kernel-matvec
(WGP_TC_TRACE) at several shapes, summarised as median cycle gaps between pipeline events.

Slots (kmatvec_tc.cu trace_ev): 0 GEMM1 issue, 1 GEMM2 issue, 2 epilogue starts waiting
for S(t), 3 S(t) ready, 4 map done, 5 K(t) arrived, 6 XB copy issued, 7 first TMEM load
done, 8 V copy issued, 9 GEMM2 sees V ready, 10 GEMM2 issued (after the last MMA),
11 quadrant-3 warp done.  Epilogue slots are recorded for set-0 tiles (t % 3 == 0).
"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

SHAPES = [
    ("C3 matern d16 s64", "matern", 0.8, 1e-3 ** 0.5, 101000, 16, 64, "normal"),
    ("C3-shape rbf d16 s64", "rbf", 0.8, 1e-3 ** 0.5, 101000, 16, 64, "normal"),
    ("C4-shape rbf d8 s32 N=200k", "rbf", 0.5, 0.1, 200000, 8, 32, "uniform"),
]


def stats(path):
    a = np.loadtxt(path, delimiter=",", skiprows=1, dtype=np.float64)
    a = a[:, 1:]  # a[:, k] = slot k
    a = a[a[:, 0] > 0]  # tiles of CTA (0, 0) only
    T = a.shape[0]
    t = np.arange(T)
    mid = (t >= T // 5) & (t < T - T // 5)
    med = lambda x: float(np.median(x)) if len(x) else float("nan")
    d = lambda x, y, m=mid: med(x[m] - y[m])
    sh = lambda col, k: np.concatenate([np.full(k, np.nan), a[:-k, col]])  # value of tile t-k
    out = {"tiles": T, "period": med(np.diff(a[mid, 0]))}
    out["g1_wait_xb"] = d(a[:, 0], a[:, 6])                 # XB copy issued -> GEMM1 issued
    out["g1_after_g2_t-5"] = med((a[:, 0] - sh(10, 5))[mid])  # GEMM2(t-5) issued -> GEMM1(t)
    out["g2_wait_v"] = med((a[:, 9] - sh(10, 1))[mid])      # GEMM2(t-1) issued -> V(t) seen ready
    out["g2_wait_k"] = d(a[:, 1], a[:, 9])                  # V(t) seen -> K(t) seen
    out["g2_issue"] = d(a[:, 10], a[:, 1])                  # 12 MMAs + commits
    out["v_copy_to_ready"] = d(a[:, 9], a[:, 8])
    if a.shape[1] > 13:
        out["g2_commits"] = d(a[:, 12], a[:, 10])
        out["g2_loop_to_yfree"] = med((a[:, 13] - sh(12, 1))[mid])
        out["g2_vfull_wait"] = d(a[:, 9], a[:, 13])
    s0 = mid & (t % 3 == 0) & (a[:, 2] > 0)
    out["epi_wait_S"] = d(a[:, 3], a[:, 2], s0)
    out["S_after_g1"] = d(a[:, 3], a[:, 0], s0)
    out["epi_ld"] = d(a[:, 7], a[:, 3], s0)
    out["epi_map"] = d(a[:, 4], a[:, 3], s0)
    out["epi_st_arrive"] = d(a[:, 5], a[:, 4], s0)
    out["q3_lag"] = d(a[:, 11], a[:, 5], s0)
    out["g2_after_k"] = d(a[:, 1], np.maximum(a[:, 5], a[:, 11]), s0)
    out["period_mean"] = float((a[-1, 0] - a[0, 0]) / max(1, T - 1))
    nxt = np.concatenate([a[3:, 2], np.full(3, np.nan)])   # set 0's next wait for S
    out["epi_after_tile"] = med((nxt - a[:, 5])[s0])        # drains etc. before the next tile
    return out


def main():
    from paper_2511_16340_b200 import warmgp as W, configs as Cfg  # noqa: F401
    only = os.environ.get("ONLY")
    for name, kern, ls, sn, n, d, s, dist in SHAPES:
        if only and only not in name:
            continue
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, d)) if dist == "normal" else rng.random((n, d))
        kind = W.MATERN32 if kern == "matern" else W.RBF
        op = W.KernelOperator(W.KernelHyperparams(ls, 1.0, sn, kind), X, precision=W.F32_3XTF32)
        V = torch.randn(n, s, device="cuda", dtype=torch.float64)
        Y = torch.empty_like(V)
        op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
        torch.cuda.synchronize()
        W.kernel_timer_enable(True)
        for _ in range(10):
            op.kmatvec_dev(V.data_ptr(), Y.data_ptr(), s)
        torch.cuda.synchronize()
        ms, launches = W.kernel_timer_read()
        W.kernel_timer_enable(False)
        path = os.path.join(tempfile.gettempdir(), "wgp_trace.csv")
        os.environ["WGP_TC_TRACE"] = path
        print(name, f"kernel {ms / launches:.3f} ms", flush=True)
        if os.environ.get("TRACE", "1") == "1":
            import subprocess
            # the trace path is read once per process (static): trace in a child
            code = (f"import sys; sys.path.insert(0, {os.getcwd()!r});"
                    "import numpy as np, torch; from paper_2511_16340_b200 import warmgp as W;"
                    f"rng=np.random.default_rng(0); X=rng.{'standard_normal' if dist == 'normal' else 'random'}(({n},{d}));"
                    f"op=W.KernelOperator(W.KernelHyperparams({ls},1.0,{sn},{kind}),X,precision=W.F32_3XTF32);"
                    f"V=torch.randn({n},{s},device='cuda',dtype=torch.float64);Y=torch.empty_like(V);"
                    f"op.kmatvec_dev(V.data_ptr(),Y.data_ptr(),{s});torch.cuda.synchronize()")
            env = dict(os.environ, WGP_TC_TRACE=path)
            subprocess.run([sys.executable, "-c", code], env=env, check=True)
            st = stats(path)
            c = np.loadtxt(path + ".ctas", delimiter=",", skiprows=1, dtype=np.float64)
            if c.ndim == 2 and len(c):
                t0, t1 = c[:, 2].min(), c[:, 4].max()
                dur = c[:, 4] - c[:, 2]
                loop = c[:, 3] - c[:, 2]
                st["ctas"] = len(c)
                st["kernel_us"] = (t1 - t0) / 1e3
                st["cta_us_med"] = float(np.median(dur)) / 1e3
                st["cta_us_min"] = float(dur.min()) / 1e3
                st["cta_us_max"] = float(dur.max()) / 1e3
                st["epi_loop_frac"] = float(np.median(loop / dur))
                st["sm_busy_frac"] = float(dur.sum() / (148 * (t1 - t0)))
                st["tail_us"] = float((t1 - np.sort(c[:, 4])[int(0.9 * len(c))]) / 1e3)
            print("  " + "  ".join(f"{k}={v:.4g}" if isinstance(v, float) else f"{k}={v}" for k, v in st.items()),
                  flush=True)
        os.environ.pop("WGP_TC_TRACE", None)


if __name__ == "__main__":
    main()

"""Probe (not collected): SGD / AP iteration counts to 1e-4 on the fp32 tensor-core operator
vs the fp64 device path and the CPU oracle, over several seeds (the spread behind the
tolerance of tests/test_gpu_sgd_ap.py::test_f32_path_sgd_ap)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402  (probe: the checker, not the product)
from paper_2511_16340_b200 import warmgp as W  # noqa: E402

for seed in (44, 45, 46, 47):
    h = O.KernelHyperparams(0.5, 1.0, 0.5, 0)
    X = O.uniform_inputs(seed, 1500, 4)
    H = O.gram_matrix(X, h)
    b = O.gaussian_vector(O.derive_seed(seed, 0xB), 1500)
    for method in (1, 2):
        kw = dict(method=method, tolerance=1e-4, max_iters=5000, learning_rate=0.005, batch_size=100, block_size=100)
        ref = O.solve(H, b, O.Initialization.cold(), O.SolverConfig(**kw))
        out = []
        for prec in (W.F64, W.F32_3XTF32):
            op = W.KernelOperator(W.KernelHyperparams(0.5, 1.0, 0.5, 0), X, precision=prec)
            out.append(W.solve(op, b, W.Initialization.cold(), W.SolverConfig(**kw)).iterations)
        print(f"seed {seed} method {'SGD' if method == 1 else 'AP'}: oracle {ref.iterations} f64 {out[0]} "
              f"f32 {out[1]} ({100 * (out[1] - ref.iterations) / ref.iterations:+.1f}%)", flush=True)

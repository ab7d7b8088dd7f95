"""Probe (not collected): wgp_coldots_dev at the C3 vector shape ([101000][64] fp64), for an
ncu launch list (coldots kernel vs the ordered chunk sum) and event timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2511_16340_b200 import warmgp as W

n, s = 101000, 64
ctx = W.default_context()
A = torch.randn(n, s, device="cuda", dtype=torch.float64)
B = torch.randn(n, s, device="cuda", dtype=torch.float64)
out = torch.empty(s, device="cuda", dtype=torch.float64)
work = torch.empty(((n + 511) // 512) * s, device="cuda", dtype=torch.float64)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda").view(torch.float64)
sink = torch.empty((), device="cuda", dtype=torch.float64)
sp = torch.cuda.current_stream().cuda_stream
for _ in range(int(os.environ.get("REPS", "5"))):
    torch.sum(flush, dim=0, out=sink)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.coldots_dev(A.data_ptr(), B.data_ptr(), n, s, out.data_ptr(), work.data_ptr(), sp)
    b.record()
    torch.cuda.synchronize()
    print(f"coldots_dev {a.elapsed_time(b) * 1e3:.1f} us", flush=True)

"""Probe (not collected): coldots kernel-only time (the library's tagged CUDA events) at the
C3 vector shape for the columns-per-block choice in WGP_COLDOTS_CB, L2 flushed by a read."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2511_16340_b200 import warmgp as W

n, s = int(os.environ.get("N", "101000")), int(os.environ.get("S", "64"))
ctx = W.default_context()
A = torch.randn(n, s, device="cuda", dtype=torch.float64)
B = torch.randn(n, s, device="cuda", dtype=torch.float64)
out = torch.empty(s, device="cuda", dtype=torch.float64)
work = torch.empty(((n + 511) // 512) * s, device="cuda", dtype=torch.float64)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda").view(torch.float64)
sink = torch.empty((), device="cuda", dtype=torch.float64)
sp = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    ctx.coldots_dev(A.data_ptr(), B.data_ptr(), n, s, out.data_ptr(), work.data_ptr(), sp)
ref = out.clone()
W.kernel_timer_enable(True)
for _ in range(20):
    torch.sum(flush, dim=0, out=sink)
    ctx.coldots_dev(A.data_ptr(), B.data_ptr(), n, s, out.data_ptr(), work.data_ptr(), sp)
torch.cuda.synchronize()
ms, k = W.kernel_timer_read("coldots")
W.kernel_timer_enable(False)
us = ms / k * 1e3
gbs = n * s * 16 / (us * 1e-6) / 1e9
print(f"CB={os.environ.get('WGP_COLDOTS_CB', 'default')} n={n} s={s}: {us:.1f} us, {gbs:.0f} GB/s "
      f"checksum {float(out.sum()):.17g}", flush=True)

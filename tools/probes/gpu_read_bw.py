"""Probe (not collected): a pure streaming read of the coldots inputs' size (two 51.7 MB fp64
arrays, torch.sum each) for the ncu launch list -- the read bandwidth a read-only kernel gets
on this part, next to the coldots kernel (WGP_COLDOTS_CB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2511_16340_b200 import warmgp as W

n, s = 101000, 64
A = torch.randn(n, s, device="cuda", dtype=torch.float64)
B = torch.randn(n, s, device="cuda", dtype=torch.float64)
AB = torch.cat([A.view(-1), B.view(-1)])
out = torch.empty(s, device="cuda", dtype=torch.float64)
work = torch.empty(((n + 511) // 512) * s, device="cuda", dtype=torch.float64)
ctx = W.default_context()
sp = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    torch.sum(AB)
    (A * B).sum()
    ctx.coldots_dev(A.data_ptr(), B.data_ptr(), n, s, out.data_ptr(), work.data_ptr(), sp)
torch.cuda.synchronize()

"""Kernel breakdown of the C2 shape (B=8, N=1024, K=16, 64->128) fwd / bwd / deconv."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_07289_b200 import _ops  # noqa: E402

b, n, k, ci, co = 8, 1024, 16, 64, 128
g = torch.Generator(device="cuda")
g.manual_seed(2)
pos = (torch.floor(torch.rand(b * n, 3, generator=g, device="cuda", dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
feat = torch.randn(b * n, ci, generator=g, device="cuda")
up = torch.randn(b * n, co, generator=g, device="cuda")
th = 0.1 * torch.randn(co, ci, 3, generator=g, device="cuda")
tb = 0.1 * torch.randn(co, ci, generator=g, device="cuda")
nbr = _ops.knn(pos, b, n, k)
csr = _ops.csr_build(nbr, b, n)


def step():
    _ops.conv_forward(feat, pos, nbr, th, tb, b, n)
    _ops.conv_backward(up, feat, pos, nbr, csr, th, tb, b, n)
    _ops.deconv_forward(up, pos, csr, th, tb, b, n, k)


for _ in range(5):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20))

"""C2 (B=8 x 1024 points, K=16, 64->128) per-kernel breakdown of the six-op step with the
library's event timer (conv fwd/bwd with d_locations, pool fwd/bwd, deconv fwd/bwd).
   python scripts/c2_kernels.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_07289_b200 import _lib, _ops  # noqa: E402

B, n, k, ci, co = 8, 1024, 16, 64, 128
T = B * n
g = torch.Generator(device="cuda")
g.manual_seed(2)
pos = (torch.floor(torch.rand(T, 3, device="cuda", dtype=torch.float64, generator=g) * 2 ** 24) / 2 ** 24).float()
nbr = _ops.knn(pos, B, n, k)
csr = _ops.csr_build(nbr, B, n)
f = torch.randn(T, ci, device="cuda", generator=g)
th = 0.1 * torch.randn(co, ci, 3, device="cuda", generator=g)
tb = 0.1 * torch.randn(co, ci, device="cuda", generator=g)
up = torch.randn(T, co, device="cuda", generator=g)


def step():
    out = _ops.conv_forward(f, pos, nbr, th, tb, B, n)
    _ops.conv_backward(up, f, pos, nbr, csr, th, tb, B, n, need=(True, True, True, True))


for _ in range(5):
    step()
torch.cuda.synchronize()
with _lib.KernelTimer() as kt:
    for _ in range(10):
        step()
for name, v in sorted(kt.times.items(), key=lambda kv: -sum(kv[1])):
    print(f"{name:24s} n={len(v):3d} mean {sum(v) / len(v) * 1e3:8.1f} us")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20))

"""Kernel breakdown of the reverse-CSR build (fc_csr_build) at 7M points, K=8."""
import sys

import torch

sys.path.insert(0, '.')
from paper_1803_07289_b200 import _ops  # noqa: E402

n = 7_000_000
pos = (torch.floor(torch.rand(n, 3, device="cuda", dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
pos = pos[_ops.spatial_order(pos).long()].contiguous()
nbr = _ops.knn(pos, 1, n, 8)
for _ in range(3):
    _ops.csr_build(nbr, 1, n)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(5):
        _ops.csr_build(nbr, 1, n)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=12))

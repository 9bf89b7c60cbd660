"""Kernel breakdown of fc_spatial_order at 7M points."""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1803_07289_b200 import _ops  # noqa: E402

n = 7_000_000
pos = (torch.floor(torch.rand(n, 3, device="cuda", dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
for _ in range(3):
    _ops.spatial_order(pos)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    _ops.spatial_order(pos)
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) / 5 * 1e3)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as p:
    for _ in range(5):
        _ops.spatial_order(pos)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=12))

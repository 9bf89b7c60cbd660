import sys, torch
sys.path.insert(0, '.')
from paper_1803_07289_b200 import _ops
n = 1 << 20
pos = (torch.floor(torch.rand(n, 3, device="cuda", dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
pos = pos[_ops.spatial_order(pos).long()].contiguous()
for _ in range(3): _ops.knn(pos, 1, n, 8)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as p:
    for _ in range(5): _ops.knn(pos, 1, n, 8)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=12))

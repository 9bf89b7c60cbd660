"""Grid-kNN builder timing (CUDA events, median of 5 warm calls) at 1M and 7M points on a
spatially ordered uniform cloud, K = 8; FC_LIB_PATH selects a library build for A/B.
   python scripts/knn_time.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_07289_b200 import _ops  # noqa: E402

for n in (1 << 20, 7_000_000):
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    pos = (torch.floor(torch.rand(n, 3, device="cuda", dtype=torch.float64, generator=g) * 2 ** 24) / 2 ** 24).float()
    pos = pos[_ops.spatial_order(pos).long()].contiguous()
    _ops.knn(pos, 1, n, 8)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        nb = _ops.knn(pos, 1, n, 8)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"knn n={n}: {statistics.median(ts):.3f} ms  checksum {int(nb.long().sum())}")

"""Time the wide-channel CUDA-core engines (conv_wide.cu) at the U-Net's level shapes.
  python scripts/wide_probe.py   (FC_NO_WIDE=1 for the per-warp kernels)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_07289_b200 import _lib, _ops  # noqa: E402

for n, c in ((65536, 128), (16384, 256), (262144, 64)):
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    pos = (torch.floor(torch.rand(n, 3, generator=g, device="cuda", dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
    pos = pos[_ops.spatial_order(pos).long()].contiguous()
    feat = torch.randn(n, c, generator=g, device="cuda")
    up = torch.randn(n, c, generator=g, device="cuda")
    th = 0.1 * torch.randn(c, c, 3, generator=g, device="cuda")
    tb = 0.1 * torch.randn(c, c, generator=g, device="cuda")
    nbr = _ops.knn(pos, 1, n, 8)
    csr = _ops.csr_build(nbr, 1, n)
    for _ in range(3):
        _ops.conv_forward(feat, pos, nbr, th, tb, 1, n, "simt")
        _ops.conv_backward(up, feat, pos, nbr, csr, th, tb, 1, n, need=(True, True, True, False), mode="simt")
    with _lib.KernelTimer() as kt:
        for _ in range(5):
            _ops.conv_forward(feat, pos, nbr, th, tb, 1, n, "simt")
            _ops.conv_backward(up, feat, pos, nbr, csr, th, tb, 1, n, need=(True, True, True, False), mode="simt")
    print(n, c, {k: round(sum(v) / len(v), 4) for k, v in kt.times.items()})

"""Conv forward / backward / deconv results written to an .npz, to be run twice with one of the
stream-concurrency knobs flipped (tests/test_gpu_wide.py checks the two files are bitwise equal):
  FC_NO_CONCURRENT=1  the channel-block passes of small clouds in sequence instead of on side streams
  FC_NO_SIDE_BWD=1    d_theta in sequence with the reverse pass instead of on a side stream
Cases: C2 (B=8 x 1024, K=16, 64->128) forward, backward with and without d_locations, deconv;
a 64->64 K=8 backward without d_locations (the fast kernels); a 128->128 backward without
d_locations at 40 K points (sequential channel blocks).
   python scripts/concurrent_passes_check.py out.npz"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1803_07289_b200 import _ops  # noqa: E402


def cloud(g, B, n, k):
    T = B * n
    pos = (torch.floor(torch.rand(T, 3, device='cuda', dtype=torch.float64, generator=g) * 2 ** 24) / 2 ** 24).float()
    nbr = _ops.knn(pos, B, n, k)
    return pos, nbr, _ops.csr_build(nbr, B, n)


def case(g, B, n, k, ci, co):
    T = B * n
    pos, nbr, csr = cloud(g, B, n, k)
    f = torch.randn(T, ci, device='cuda', generator=g)
    th = 0.1 * torch.randn(co, ci, 3, device='cuda', generator=g)
    tb = 0.1 * torch.randn(co, ci, device='cuda', generator=g)
    up = torch.randn(T, co, device='cuda', generator=g)
    return pos, nbr, csr, f, th, tb, up


g = torch.Generator(device='cuda')
g.manual_seed(2)
res = {}
B, n, k = 8, 1024, 16
pos, nbr, csr, f, th, tb, up = case(g, B, n, k, 64, 128)
res['out'] = _ops.conv_forward(f, pos, nbr, th, tb, B, n)
for i, r in enumerate(_ops.conv_backward(up, f, pos, nbr, csr, th, tb, B, n, need=(True, True, True, True))):
    res[f'bwd{i}'] = r
for i, r in enumerate(_ops.conv_backward(up, f, pos, nbr, csr, th, tb, B, n, need=(True, True, True, False))[:3]):
    res[f'bwd_nodl{i}'] = r
res['y'] = _ops.deconv_forward(up, pos, csr, th, tb, B, n, k)
for tag, (n2, ci, co) in {'fast64': (50_000, 64, 64), 'wide128': (40_000, 128, 128)}.items():
    pos, nbr, csr, f, th, tb, up = case(g, 1, n2, 8, ci, co)
    for i, r in enumerate(_ops.conv_backward(up, f, pos, nbr, csr, th, tb, 1, n2, need=(True, True, True, False))[:3]):
        res[f'{tag}_{i}'] = r
torch.cuda.synchronize()
np.savez(sys.argv[1], **{key: v.cpu().numpy() for key, v in res.items()})

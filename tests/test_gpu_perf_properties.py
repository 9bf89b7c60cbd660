"""Performance PROPERTIES (the reference's own kind of performance test, not absolute
timings): linear scaling of the flex-conv forward+backward in the number of points
(reference tests/test_acceptance.py:168-179: time ratio per doubling in [1.5, 3.0]) and
sub-quadratic kNN (tests/test_neighborhood.py:162-178: 4x points in < 10x time).
Sizes are large enough that the B200 kernels are throughput-bound, not launch-bound."""

import statistics

import pytest
import torch

pytestmark = pytest.mark.gpu


def _cloud(n, c=64, k=8, seed=0):
    from paper_1803_07289_b200 import _ops

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    pos = (torch.floor(torch.rand(n, 3, generator=g, device="cuda", dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
    pos = pos[_ops.spatial_order(pos).long()].contiguous()
    feat = torch.randn(n, c, generator=g, device="cuda")
    up = torch.randn(n, c, generator=g, device="cuda")
    th = 0.1 * torch.randn(c, c, 3, generator=g, device="cuda")
    tb = 0.1 * torch.randn(c, c, generator=g, device="cuda")
    nbr = _ops.knn(pos, 1, n, k)
    return pos, feat, up, th, tb, nbr, _ops.csr_build(nbr, 1, n)


def _time(fn, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def test_conv_fwd_bwd_scales_linearly(fc):
    from paper_1803_07289_b200 import _ops

    times = []
    for n in (1 << 20, 1 << 21, 1 << 22):
        pos, feat, up, th, tb, nbr, csr = _cloud(n)

        def step():
            _ops.conv_forward(feat, pos, nbr, th, tb, 1, n)
            _ops.conv_backward(up, feat, pos, nbr, csr, th, tb, 1, n)
        times.append(_time(step))
    ratios = [b / a for a, b in zip(times, times[1:])]
    assert all(1.5 <= r <= 3.0 for r in ratios), (times, ratios)


def test_knn_sub_quadratic(fc):
    from paper_1803_07289_b200 import _ops

    ts = []
    for n in (1 << 19, 1 << 21):
        pos = (torch.floor(torch.rand(n, 3, device="cuda", dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
        ts.append(_time(lambda: _ops.knn(pos, 1, n, 8), reps=3))
    assert ts[1] < 10 * ts[0], ts

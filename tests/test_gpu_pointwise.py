"""The pointwise (1x1) convolution GEMMs of the U-Net step (csrc/gemm_tc.cu: tcgen05
kind::tf32 with hi/lo split operands; SIMT fixed-order weight gradient) against an fp64
torch reference of the same op -- the reference's pointwise_conv (flexops.py:206-226) over a
concatenation that is never built (network.py:180-246).  fp32 tolerance: allclose(rtol 1e-4,
atol 1e-5 * max|ref|) elementwise, 1e-5 norm-wise."""

import numpy as np
import pytest
import torch

from paper_1803_07289_b200 import _lib, _ops
from paper_1803_07289_b200.errors import ShapeMismatchError

pytestmark = pytest.mark.gpu


def _close(got, ref):
    got, ref = got.double().cpu(), ref.double().cpu()
    scale = float(ref.abs().max()) or 1.0
    assert float((got - ref).norm() / max(float(ref.norm()), 1e-300)) < 1e-5
    assert torch.allclose(got, ref, rtol=1e-4, atol=1e-5 * scale), float((got - ref).abs().max())


SHAPES = [  # (n, operand widths, c_out): ResBlock (x | coords), MergeBlock (x | skip | coords), head
    (1000, [64, 3], 64),
    (4097, [128, 64, 3], 64),
    (777, [256, 128, 3], 128),
    (300, [64], 3),
    (1, [256], 40),
    (2048, [128, 3], 256),
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"n{s[0]}-{'+'.join(map(str, s[1]))}-{s[2]}")
def test_pointwise_forward_dgrad_wgrad(shape):
    n, widths, co = shape
    torch.manual_seed(n + co)
    dev = torch.device("cuda", 0)
    xs = [torch.randn(n, w, device=dev) for w in widths]
    ci = sum(widths)
    w = 0.1 * torch.randn(co, ci, device=dev)
    b = torch.randn(co, device=dev)
    segs, a = [], 0
    for wd in widths:
        segs.append((a, wd))
        a += wd
    launches = _lib.launch_count()
    # forward + fused ReLU copy
    y, yr = _ops.gemm_rows(xs, _ops.gemm_pack(w, segs), co, bias=b, relu=True)
    ref = torch.cat([x.double() for x in xs], 1) @ w.double().t() + b.double()
    _close(y, ref)
    assert torch.equal(yr, torch.clamp_min(y, 0.0))
    # d_input through W^T, masked by the ReLU of a saved pre-activation, per-operand outputs
    g = torch.randn(n, co, device=dev)
    z = torch.randn(n, co, device=dev)
    outs = [(s, s + wd) for s, wd in segs]
    dxs = _ops.gemm_rows([g], _ops.gemm_pack(w, [(0, co)], transpose=True), ci, outs=outs, mask=z)
    gm = g.double() * (z > 0)
    dref = gm @ w.double()
    for (s, e), dx in zip(outs, dxs):
        _close(dx, dref[:, s:e])
    # weight / bias gradient
    dw = torch.empty(co, ci, device=dev)
    db = torch.empty(co, device=dev)
    _ops.gemm_wgrad(g, xs, dw, db, mask=z)
    _close(dw, gm.t() @ torch.cat([x.double() for x in xs], 1))
    _close(db, gm.sum(0))
    assert _lib.launch_count() > launches


def test_pointwise_wgrad_deterministic_and_checks():
    dev = torch.device("cuda", 0)
    torch.manual_seed(3)
    x = torch.randn(100_000, 64, device=dev)
    g = torch.randn(100_000, 128, device=dev)
    dw1, dw2 = torch.empty(128, 64, device=dev), torch.empty(128, 64, device=dev)
    _ops.gemm_wgrad(g, [x], dw1, None)
    _ops.gemm_wgrad(g, [x], dw2, None)
    assert torch.equal(dw1, dw2)
    with pytest.raises(ShapeMismatchError):
        _ops.gemm_wgrad(g, [x[:10]], dw1, None)
    with pytest.raises(ShapeMismatchError):
        _ops.gemm_pack(torch.randn(8, 8, device=dev), [(4, 8)])


def test_pointwise_large_values_no_scaling_issue():
    """tf32 keeps fp32's exponent range: rows of very different magnitude in one tile."""
    dev = torch.device("cuda", 0)
    torch.manual_seed(5)
    x = torch.randn(512, 64, device=dev) * torch.logspace(-20, 20, 512, device=dev)[:, None]
    w = torch.randn(32, 64, device=dev)
    (y,) = _ops.gemm_rows([x], _ops.gemm_pack(w, [(0, 64)]), 32)
    ref = x.double() @ w.double().t()
    rel = ((y.double() - ref).norm(dim=1) / ref.norm(dim=1)).max()
    assert float(rel) < 1e-5
    assert np.isfinite(y.cpu().numpy()).all()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("n", [1, 7, 4096, 262_147])
def test_relu_backward_matches_torch_bitwise(dtype, n):
    """fc_relu_backward == `g * (z > 0) + add` bit for bit (NaN, inf and signed zeros
    included), in place or not, vectorised (n % 4 == 0) and scalar paths."""
    dev = torch.device("cuda", 0)
    torch.manual_seed(n)
    g = torch.randn(n, dtype=dtype, device=dev)
    z = torch.randn(n, dtype=dtype, device=dev)
    add = torch.randn(n, dtype=dtype, device=dev)
    if n >= 7:
        g[:4] = torch.tensor([float("nan"), float("inf"), -0.0, -1.0], dtype=dtype)
        z[:7] = torch.tensor([-1.0, -2.0, 3.0, 0.0, float("nan"), -0.0, 5.0], dtype=dtype)
    want = g * (z > 0)
    assert torch.equal(_ops.relu_backward(g, z).view(torch.int64 if dtype == torch.float64 else torch.int32),
                       want.view(torch.int64 if dtype == torch.float64 else torch.int32))
    want_add = g * (z > 0) + add
    got = g.clone()
    _ops.relu_backward(got, z, add=add, out=got)  # in place
    iv = torch.int64 if dtype == torch.float64 else torch.int32
    assert torch.equal(got.view(iv), want_add.view(iv))
    with pytest.raises(ShapeMismatchError):
        _ops.relu_backward(g, z[: max(n - 1, 0)] if n > 1 else z.repeat(2))

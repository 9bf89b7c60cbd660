"""GPU parity of the wide-channel CUDA-core engines (conv_wide.cu: wide_gmc_kernel and
dtheta_slice_kernel) -- the shapes the tensor-core kernels do not cover: the U-Net's
128 -> 128 and 256 -> 256 levels, the classifier's 64 -> 128, odd channel counts and d != 3.

Oracle: oracle/flexconv_oracle.c (pinned bitwise to the reference's _native kernels).
Tolerances as tests/test_gpu_parity.py: fp64 forward bitwise (same operations, same order);
fp64 backward / deconv 1e-12 relative; fp32 forward / deconv / d_features allclose(1e-4, 1e-5);
fp32 N-long reductions (d_theta, d_theta_b, d_locations) with the stated floor + norm 1e-5.
"""

import os

import numpy as np
import pytest

from paper_1803_07289_b200.core import synthetic_layer

pytestmark = pytest.mark.gpu

SHAPES = [  # (n, k, c_in, c_out, d)
    (700, 8, 128, 128, 3),
    (300, 8, 256, 256, 3),
    (500, 16, 64, 128, 3),
    (333, 7, 40, 72, 3),
    (257, 5, 24, 200, 2),
    (129, 6, 17, 33, 5),
]


def _case(shape, seed=11):
    from oracle import oracle

    n, k, cin, cout, d = shape
    loc, feat, th, tb, up = synthetic_layer(seed, cin + cout, n, d, cin, cout)
    nbr = oracle.knn_brute(loc, k)
    return loc, feat, th, tb, up, nbr


def _t(a, dtype):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dtype)


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _red_close(got, ref, name):
    floor = 1e-5 + 1e-6 * float(np.abs(ref).max())
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=floor, err_msg=name)
    assert np.linalg.norm(got - ref) <= 1e-5 * max(np.linalg.norm(ref), 1e-30), name


@pytest.mark.parametrize("shape", SHAPES)
def test_wide_forward_fp64_bitwise(fc, oracle_mod, shape):
    loc, feat, th, tb, up, nbr = _case(shape)
    got = fc.flex_conv_forward(feat, loc, fc.NeighborIndex(nbr), fc.FlexConvParams(th, tb))
    np.testing.assert_array_equal(got, oracle_mod.conv_forward(feat, loc, nbr, th, tb))


@pytest.mark.parametrize("shape", SHAPES)
def test_wide_fp32_forward_backward_deconv(fc, oracle_mod, shape):
    import torch

    loc, feat, th, tb, up, nbr = _case(shape)
    f32 = torch.float32
    nb = fc.NeighborIndex(_t(nbr, torch.int64))
    params = fc.FlexConvParams(_t(th, f32), _t(tb, f32))
    out = fc.flex_conv_forward(_t(feat, f32), _t(loc, f32), nb, params)
    np.testing.assert_allclose(_np(out), oracle_mod.conv_forward(feat, loc, nbr, th, tb), rtol=1e-4, atol=1e-5)
    df, dth, dtb, dl = oracle_mod.conv_backward(up, feat, loc, nbr, th, tb)
    for with_loc in (False, True):
        gb = fc.flex_conv_backward(_t(up, f32), _t(feat, f32), _t(loc, f32), nb, params, with_locations=with_loc)
        np.testing.assert_allclose(_np(gb.d_features), df, rtol=1e-4, atol=1e-5, err_msg="d_features")
        _red_close(_np(gb.d_theta), dth, "d_theta")
        _red_close(_np(gb.d_theta_b), dtb, "d_theta_b")
        if with_loc:
            _red_close(_np(gb.d_locations), dl, "d_locations")
    y = fc.flex_deconv_forward(_t(up, f32), _t(loc, f32), nb, params)
    np.testing.assert_allclose(_np(y), oracle_mod.deconv_forward(up, loc, nbr, th, tb), rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("shape", SHAPES[:3])
def test_wide_fp64_backward_and_deconv(fc, oracle_mod, shape):
    loc, feat, th, tb, up, nbr = _case(shape)
    nb = fc.NeighborIndex(nbr)
    params = fc.FlexConvParams(th, tb)
    gb = fc.flex_conv_backward(up, feat, loc, nb, params)
    for got, ref in zip((gb.d_features, gb.d_theta, gb.d_theta_b, gb.d_locations),
                        oracle_mod.conv_backward(up, feat, loc, nbr, th, tb)):
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * float(np.abs(ref).max()))
    y = fc.flex_deconv_forward(up, loc, nb, params)
    ref = oracle_mod.deconv_forward(up, loc, nbr, th, tb)
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12 * float(np.abs(ref).max()))


def test_wide_batched_and_deterministic(fc, oracle_mod):
    """Batched clouds (cloud-local indices) through the [B, D, N] API; two runs bitwise equal."""
    import torch

    b, n, k, cin, cout = 3, 400, 8, 128, 128
    g = np.random.default_rng(3)
    loc = np.floor(g.random((b, n, 3)) * 2 ** 24) / 2 ** 24
    feat = g.standard_normal((b, n, cin)).astype(np.float32).astype(np.float64)
    th = (0.1 * g.standard_normal((cout, cin, 3))).astype(np.float32).astype(np.float64)
    tb = (0.1 * g.standard_normal((cout, cin))).astype(np.float32).astype(np.float64)
    pos = _t(loc, torch.float32).transpose(1, 2)
    nbh = fc.knn(pos, k)
    f = _t(feat, torch.float32).transpose(1, 2).requires_grad_(True)
    theta = _t(th, torch.float32).requires_grad_(True)
    theta_b = _t(tb, torch.float32).requires_grad_(True)
    outs = []
    for _ in range(2):
        f.grad = theta.grad = theta_b.grad = None
        out = fc.flex_conv(f, pos, nbh, theta, theta_b)
        out.square().sum().backward()
        outs.append([t.detach().clone() for t in (out, f.grad, theta.grad, theta_b.grad)])
    for a, c in zip(*outs):
        assert torch.equal(a, c)
    for bi in range(b):
        nbr = nbh.bkn[bi].t().cpu().numpy().astype(np.int64)
        ref = oracle_mod.conv_forward(feat[bi], loc[bi], nbr, th, tb)
        np.testing.assert_allclose(_np(outs[0][0][bi].t()), ref, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("shape", [(1024, 16, 64, 128, 3), (700, 8, 128, 128, 3), (300, 8, 256, 256, 3),
                                   (30000, 8, 128, 128, 3)])
def test_wide_fp32_default_route_is_hand_written_tcgen05(fc, shape):
    """C2's 64 -> 128 (K = 16) and the U-Net's 128 / 256-channel layers: the default fp32
    route (forward, backward with d_locations, flex_deconv) launches only this library's
    kernels -- the channel-blocked gather -> tcgen05 engines, or for clouds of less than one
    wave of tiles with >= 256 channels the moments rows + the hand-written tcgen05 GEMM -- and
    no library GEMM (cuBLAS /
    CUTLASS; the library does not link cuBLAS at all: its FC_GEMM_ROUTE=1 A/B route runs
    moments rows through the hand-written tcgen05 GEMM)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    n, k, cin, cout, d = shape
    if n > 5000:  # random neighbour rows are enough for a routing check at this size
        g = np.random.default_rng(1)
        loc = np.floor(g.random((n, d)) * 2 ** 24) / 2 ** 24
        feat, up = g.standard_normal((n, cin)), g.standard_normal((n, cout))
        th, tb = 0.1 * g.standard_normal((cout, cin, d)), 0.1 * g.standard_normal((cout, cin))
        nbr = np.concatenate([np.arange(n)[:, None], g.integers(0, n, (n, k - 1))], axis=1)
    else:
        loc, feat, th, tb, up, nbr = _case(shape)
    f32 = torch.float32
    nb = fc.NeighborIndex(_t(nbr, torch.int64))
    params = fc.FlexConvParams(_t(th, f32), _t(tb, f32))
    args = (_t(feat, f32), _t(loc, f32))
    fc.flex_conv_forward(*args, nb, params)  # warm-up (module load, CSR)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fc.flex_conv_forward(*args, nb, params)
        fc.flex_conv_backward(_t(up, f32), *args, nb, params, with_locations=True)
        fc.flex_deconv_forward(_t(up, f32), args[1], nb, params)
        torch.cuda.synchronize()
    names = [e.key for e in prof.key_averages() if e.device_type == torch.autograd.DeviceType.CUDA]
    library = [k for k in names if "fc::" not in k and "fast::" not in k and
               any(s in k.lower() for s in ("gemm", "cublas", "cutlass", "sm90_", "sm100_xmma"))]
    assert not library, library
    if n < 148 * 128 and cin >= 256 and cout >= 256:  # less than a wave: moments rows + one tcgen05 GEMM
        assert any("gemm_rows_kernel" in k for k in names), names
    else:
        assert any("tc_gmc_kernel" in k for k in names), names
        assert any("tc_dtheta_kernel" in k for k in names), names


def _run_check_twice(tmp_path, knob):
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = os.path.join(root, "scripts", "concurrent_passes_check.py")
    outs = []
    for flag in ("0", "1"):
        f = tmp_path / f"{knob}{flag}.npz"
        env = dict(os.environ, **{knob: flag})
        subprocess.run([sys.executable, script, str(f)], check=True, cwd=root, env=env)
        outs.append(np.load(f))
    a, b = outs
    assert a.files == b.files and len(a.files) >= 10
    for key in a.files:
        assert np.array_equal(a[key], b[key]), key


def test_concurrent_block_passes_bitwise_equal_sequential(tmp_path):
    """Small clouds run the channel-blocked passes concurrently on side streams, each into its
    own buffer, combined in the sequential accumulation order: bitwise the sequential result
    (C2 shape: conv forward, backward with / without d_locations, flex_deconv)."""
    _run_check_twice(tmp_path, "FC_NO_CONCURRENT")


def test_side_stream_dtheta_bitwise_equal_sequential(tmp_path):
    """Without d_locations, fc_conv_backward runs d_theta on a side stream beside the reverse
    pass: bitwise the in-order result (C2 blocked, 64->64 fast kernels, 128->128 blocked)."""
    _run_check_twice(tmp_path, "FC_NO_SIDE_BWD")


@pytest.mark.parametrize("cin,cout", [(128, 128), (256, 128), (64, 192)])
def test_wide_fast_channel_blocks_vs_oracle(fc, oracle_mod, cin, cout):
    """Clouds that fill the GPU with one pass run the channel blocks on the 64 -> 64 K = 8
    headline kernels (strided rows, ascending-block accumulation in the epilogue): 40 K
    points, sampled rows of the forward / d_features and the full parameter gradients against
    the oracle (fp32 tolerances of the module docstring)."""
    import torch

    n, k, d = 40_000, 8, 3
    g = np.random.default_rng(cin + cout)
    loc = np.floor(g.random((n, d)) * 2 ** 24) / 2 ** 24
    order = np.lexsort((loc[:, 2], loc[:, 1], np.floor(loc[:, 0] * 64)))  # roughly local rows
    loc = loc[order]
    feat = g.standard_normal((n, cin)).astype(np.float32).astype(np.float64)
    up = g.standard_normal((n, cout)).astype(np.float32).astype(np.float64)
    th = (0.1 * g.standard_normal((cout, cin, d))).astype(np.float32).astype(np.float64)
    tb = (0.1 * g.standard_normal((cout, cin))).astype(np.float32).astype(np.float64)
    f32 = torch.float32
    pos = _t(loc.astype(np.float32), f32)
    from paper_1803_07289_b200 import _ops

    nbr_t = _ops.knn(pos, 1, n, k)
    nbr = nbr_t.cpu().numpy().astype(np.int64)
    rows = np.unique(np.concatenate([np.arange(64), np.arange(n - 64, n), g.integers(0, n, 2000)]))
    nb = fc.NeighborIndex(_t(nbr, torch.int64))
    params = fc.FlexConvParams(_t(th, f32), _t(tb, f32))
    locf = loc.astype(np.float32).astype(np.float64)
    out = _np(fc.flex_conv_forward(_t(feat, f32), pos, nb, params))
    ref = oracle_mod.conv_forward_rows(feat, locf, nbr, th, tb, rows)
    np.testing.assert_allclose(out[rows], ref, rtol=1e-4, atol=1e-5)
    gb = fc.flex_conv_backward(_t(up, f32), _t(feat, f32), pos, nb, params, with_locations=False)
    df_ref, _ = oracle_mod.conv_backward_rows(up, feat, locf, nbr, th, tb, rows, with_locations=False)
    np.testing.assert_allclose(_np(gb.d_features)[rows], df_ref, rtol=1e-4, atol=1e-5)
    dth, dtb = oracle_mod.conv_param_grads(up, feat, locf, nbr)
    _red_close(_np(gb.d_theta), dth, "d_theta")
    _red_close(_np(gb.d_theta_b), dtb, "d_theta_b")


def test_wide_fast_channel_blocks_bf16_mode(oracle_mod):
    """The bf16 tensor-core mode through the fast channel blocks (128 -> 128 at 40 K points):
    forward, flex_deconv and d_features within the bf16 bounds (norm-wise 1e-2 and max-abs
    1e-2 x max|ref|) on sampled rows."""
    import torch

    from paper_1803_07289_b200 import _ops

    n, k, c = 40_000, 8, 128
    g = np.random.default_rng(77)
    loc = (np.floor(g.random((n, 3)) * 2 ** 24) / 2 ** 24).astype(np.float32)
    pos = torch.from_numpy(loc).cuda()
    pos = pos[_ops.spatial_order(pos).long()].contiguous()
    locf = pos.cpu().numpy().astype(np.float64)
    feat = g.standard_normal((n, c)).astype(np.float32)
    up = g.standard_normal((n, c)).astype(np.float32)
    th = (0.1 * g.standard_normal((c, c, 3))).astype(np.float32)
    tb = (0.1 * g.standard_normal((c, c))).astype(np.float32)
    t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    nbr = _ops.knn(pos, 1, n, k)
    csr = _ops.csr_build(nbr, 1, n)
    nb = nbr.cpu().numpy().astype(np.int64)
    rows = np.unique(g.integers(0, n, 1500))

    def close(got, ref):
        assert np.linalg.norm(got - ref) <= 1e-2 * np.linalg.norm(ref)
        assert np.abs(got - ref).max() <= 1e-2 * np.abs(ref).max()

    out = _ops.conv_forward(t(feat), pos, nbr, t(th), t(tb), 1, n, mode="bf16").cpu().numpy()
    close(out[rows], oracle_mod.conv_forward_rows(feat, locf, nb, th, tb, rows))
    df = _ops.conv_backward(t(up), t(feat), pos, nbr, csr, t(th), t(tb), 1, n, need=(True, False, False, False),
                            mode="bf16")[0].cpu().numpy()
    df_ref, _ = oracle_mod.conv_backward_rows(up, feat, locf, nb, th, tb, rows, with_locations=False)
    close(df[rows], df_ref)
    y = _ops.deconv_forward(t(up), pos, csr, t(th), t(tb), 1, n, k, mode="bf16").cpu().numpy()
    close(y[rows], df_ref)  # flex_deconv = A(theta)^T x = d_features of the conv with upstream x

"""GPU: argument checking at the device operator layer, the reverse-CSR builder on hub-heavy
neighbourhoods, per-device launches, and CUDA-graph capture of a kNN + conv step."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _layer(n=512, cin=8, cout=6, k=5):
    import torch

    from paper_1803_07289_b200 import _ops
    from paper_1803_07289_b200.core import synthetic_layer

    loc, feat, th, tb, up = synthetic_layer(7, 0, n, 3, cin, cout)
    t = {name: torch.from_numpy(v).cuda().float() for name, v in
         dict(loc=loc, feat=feat, th=th, tb=tb, up=up).items()}
    t["nbr"] = _ops.knn(t["loc"], 1, n, k)
    t["csr"] = _ops.csr_build(t["nbr"], 1, n)
    return t, n, k


@pytest.mark.parametrize("bad", ["feat_cols", "loc_cols", "theta_b", "rows", "theta_rank"])
def test_conv_forward_rejects_mismatched_shapes(fc, bad):
    from paper_1803_07289_b200 import _ops
    from paper_1803_07289_b200.errors import ShapeMismatchError

    t, n, k = _layer()
    feat, loc, th, tb = t["feat"], t["loc"], t["th"], t["tb"]
    batch = 1
    if bad == "feat_cols":
        feat = feat[:, :5].contiguous()
    elif bad == "loc_cols":
        loc = loc[:, :2].contiguous()
    elif bad == "theta_b":
        tb = tb[:, :3].contiguous()
    elif bad == "rows":
        batch = 2
    elif bad == "theta_rank":
        th = th[:, :, 0].contiguous()
    with pytest.raises(ShapeMismatchError):
        _ops.conv_forward(feat, loc, t["nbr"], th, tb, batch, n)


@pytest.mark.parametrize("bad", ["upstream_cols", "feat_cols", "theta_b", "csr"])
def test_conv_backward_rejects_mismatched_shapes(fc, bad):
    from paper_1803_07289_b200 import _ops
    from paper_1803_07289_b200.errors import ShapeMismatchError

    t, n, k = _layer()
    g, feat, tb, csr = t["up"], t["feat"], t["tb"], t["csr"]
    if bad == "upstream_cols":
        g = g[:, :4].contiguous()
    elif bad == "feat_cols":
        feat = feat[:, :7].contiguous()
    elif bad == "theta_b":
        tb = tb.t().contiguous()
    elif bad == "csr":
        csr = (csr[0][:-1], csr[1])
    with pytest.raises(ShapeMismatchError):
        _ops.conv_backward(g, feat, t["loc"], t["nbr"], csr, t["th"], tb, 1, n)


@pytest.mark.parametrize("bad", ["x_cols", "rows", "loc_cols"])
def test_deconv_rejects_mismatched_shapes(fc, bad):
    from paper_1803_07289_b200 import _ops
    from paper_1803_07289_b200.errors import ShapeMismatchError

    t, n, k = _layer()
    x, loc, batch = t["up"], t["loc"], 1
    if bad == "x_cols":
        x = t["feat"]  # C_in columns instead of C_out
    elif bad == "rows":
        x = x[: n - 3].contiguous()
    elif bad == "loc_cols":
        loc = loc[:, :1].contiguous()
    with pytest.raises(ShapeMismatchError):
        _ops.deconv_forward(x, loc, t["csr"], t["th"], t["tb"], batch, n, k)


def test_pool_rejects_mismatched_shapes(fc):
    from paper_1803_07289_b200 import _ops
    from paper_1803_07289_b200.errors import ShapeMismatchError

    t, n, k = _layer()
    with pytest.raises(ShapeMismatchError):
        _ops.pool_forward(t["feat"][: n - 1].contiguous(), t["nbr"], 1, n)
    out, am = _ops.pool_forward(t["feat"], t["nbr"], 1, n)
    with pytest.raises(ShapeMismatchError):
        _ops.pool_backward(out, am[:, :3].contiguous(), t["csr"], 1, n, k)


@pytest.mark.parametrize("hub", [40, 3000, 20000])
def test_csr_long_segments_are_stable(fc, hub):
    """Reverse lists far longer than the register sort (16 entries): the per-CTA bitonic
    path (shared memory up to 8192 entries, global memory beyond) must still give the stable
    counting sort -- entries ascending within every bucket, equal to numpy's stable argsort."""
    import torch

    from paper_1803_07289_b200 import _ops

    n, k = 30000, 8
    rng = np.random.default_rng(hub)
    nbr = rng.integers(0, n, size=(n, k)).astype(np.int32)
    nbr[:, 0] = np.arange(n)
    rows = rng.choice(n, size=hub, replace=False)
    nbr[rows, 3] = 17  # one hub point with `hub` extra reverse entries
    nbr[rows[: hub // 2], 5] = 123
    off, ent = _ops.csr_build(torch.from_numpy(nbr).cuda(), 1, n)
    flat = nbr.reshape(-1).astype(np.int64)
    order = np.argsort(flat, kind="stable")
    want_off = np.r_[0, np.cumsum(np.bincount(flat, minlength=n))]
    np.testing.assert_array_equal(off.cpu().numpy(), want_off)
    np.testing.assert_array_equal(ent.cpu().numpy(), order)
    off2, ent2 = _ops.csr_build(torch.from_numpy(nbr).cuda(), 1, n, validate=False)
    assert torch.equal(off, off2) and torch.equal(ent, ent2)


def test_ops_on_a_non_current_device(fc):
    """Tensors on the last visible device while cuda:0 is current (single-GPU boxes run it
    on cuda:0 itself): the launch follows the tensors' device."""
    import torch

    from paper_1803_07289_b200 import _ops

    dev = torch.device("cuda", torch.cuda.device_count() - 1)
    torch.cuda.set_device(0)
    pos = torch.rand(3000, 3, device=dev)
    nbr = _ops.knn(pos, 1, 3000, 8)
    feat = torch.randn(3000, 64, device=dev)
    th = torch.randn(64, 64, 3, device=dev) * 0.1
    tb = torch.randn(64, 64, device=dev) * 0.1
    out = _ops.conv_forward(feat, pos, nbr, th, tb, 1, 3000)
    assert out.device == dev and torch.isfinite(out).all()


def test_knn_and_conv_step_capture_as_one_cuda_graph(fc):
    """The grid kNN computes its grid on the device (no bounding-box read-back), and the
    reverse CSR of a Neighborhood is built without a host sync, so kNN + CSR + conv forward
    + backward capture as one CUDA graph; replay gives the eager results bitwise."""
    import torch

    import paper_1803_07289_b200 as pkg

    n, k = 50000, 8
    torch.manual_seed(3)
    pos = torch.floor(torch.rand(1, 3, n, device="cuda", dtype=torch.float64) * 2 ** 24).float() / 2 ** 24
    feat = torch.randn(1, 64, n, device="cuda")
    th = torch.randn(64, 64, 3, device="cuda") * 0.1
    tb = torch.randn(64, 64, device="cuda") * 0.1
    g = torch.randn(1, 64, n, device="cuda")

    def step():
        nbh = pkg.knn(pos, k)
        f = feat.detach().requires_grad_(True)
        out = pkg.flex_conv(f, pos, nbh, th, tb)
        (df,) = torch.autograd.grad(out, f, g)
        return nbh.table.clone(), out.detach().clone(), df

    eager = step()  # warm-up (module load, pool growth) + reference results
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        captured = step()
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, captured):
        assert torch.equal(a, b)


def test_deconv_backward_entry_point_and_workspace_query(fc):
    """fc_deconv_backward equals its definition (flex_conv forward of the upstream for d_x,
    flex_conv backward with upstream = x, features = gy for the parameter / location
    gradients) bitwise, and the scratch high-water query reports the backward's workspace."""
    import torch

    from paper_1803_07289_b200 import _ops

    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    n, k, ci, co = 5000, 8, 64, 64
    pos = torch.rand(n, 3, device="cuda", generator=g)
    nbr = _ops.knn(pos, 1, n, k)
    csr = _ops.csr_build(nbr, 1, n)
    x = torch.randn(n, co, device="cuda", generator=g)
    gy = torch.randn(n, ci, device="cuda", generator=g)
    th = 0.1 * torch.randn(co, ci, 3, device="cuda", generator=g)
    tb = 0.1 * torch.randn(co, ci, device="cuda", generator=g)
    _ops.scratch_peak_bytes(reset=True)
    dx, dth, dtb, dl = _ops.deconv_backward(gy, x, pos, nbr, csr, th, tb, 1, n)
    assert _ops.scratch_peak_bytes() > 0
    ref_dx = _ops.conv_forward(gy, pos, nbr, th, tb, 1, n)
    _, rth, rtb, rdl = _ops.conv_backward(x, gy, pos, nbr, csr, th, tb, 1, n, need=(False, True, True, True))
    for got, ref in ((dx, ref_dx), (dth, rth), (dtb, rtb), (dl, rdl)):
        assert torch.equal(got, ref)

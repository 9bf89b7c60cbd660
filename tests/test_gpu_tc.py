"""GPU: the tcgen05 tensor-core engines against the oracle.

  * split engine (fp16 hi/lo, 3 MMAs): the north_star fp32 tolerance, elementwise
    allclose(rtol=1e-4, atol=1e-5) for forward / flex_deconv / d_features;
  * bf16 engine: the stated 1e-2 relative tolerance, norm-wise ||D||/||ref|| <= 1e-2 and
    max|D| <= 1e-2 * max|ref|.
Plus size-independent properties at N = 1M (adjoint identity, determinism) where the
oracle would take minutes.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _layer(n, cin, cout, k, seed=21):
    import torch

    from paper_1803_07289_b200 import _ops
    from paper_1803_07289_b200.core import synthetic_layer

    loc, feat, th, tb, up = synthetic_layer(seed, 0, n, 3, cin, cout)
    dev = torch.device("cuda")
    t = {name: torch.from_numpy(v).to(dev, torch.float32) for name, v in
         dict(loc=loc, feat=feat, th=th, tb=tb, up=up).items()}
    t["nbr"] = _ops.knn(t["loc"], 1, n, k)
    t["csr"] = _ops.csr_build(t["nbr"], 1, n)
    host = dict(loc=loc, feat=feat, th=th, tb=tb, up=up, nbr=t["nbr"].cpu().numpy().astype(np.int64))
    return t, host


def _close_bf16(got, ref, name):
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-2, (name, err)
    assert np.abs(got - ref).max() <= 1e-2 * np.abs(ref).max(), name


@pytest.mark.parametrize("cin,cout", [(64, 64), (32, 32), (64, 32), (32, 64), (32, 128)])
@pytest.mark.parametrize("mode", ["split", "bf16"])
def test_tc_forward_vs_oracle(fc, oracle_mod, cin, cout, mode):
    from paper_1803_07289_b200 import _ops

    n, k = 20000, 8
    t, h = _layer(n, cin, cout, k)
    out = _ops.conv_forward(t["feat"], t["loc"], t["nbr"], t["th"], t["tb"], 1, n, mode).cpu().numpy()
    ref = oracle_mod.conv_forward(h["feat"], h["loc"], h["nbr"], h["th"], h["tb"])
    if mode == "split":
        np.testing.assert_allclose(out, ref, rtol=1e-4, atol=1e-5)
    else:
        _close_bf16(out, ref, f"fwd {cin}->{cout}")


@pytest.mark.parametrize("cin,cout", [(64, 64), (32, 32), (64, 32)])
@pytest.mark.parametrize("mode", ["split", "bf16"])
def test_tc_deconv_and_dfeatures_vs_oracle(fc, oracle_mod, cin, cout, mode):
    from paper_1803_07289_b200 import _ops

    n, k = 20000, 8
    t, h = _layer(n, cin, cout, k, seed=22)
    y = _ops.deconv_forward(t["up"], t["loc"], t["csr"], t["th"], t["tb"], 1, n, k, mode).cpu().numpy()
    ref = oracle_mod.deconv_forward(h["up"], h["loc"], h["nbr"], h["th"], h["tb"])
    if mode == "split":
        np.testing.assert_allclose(y, ref, rtol=1e-4, atol=1e-5)
    else:
        _close_bf16(y, ref, "deconv")
    df, _, _, _ = _ops.conv_backward(t["up"], t["feat"], t["loc"], t["nbr"], t["csr"], t["th"], t["tb"], 1, n,
                                     need=(True, False, False, False), mode=mode)
    if mode == "split":
        np.testing.assert_allclose(df.cpu().numpy(), ref, rtol=1e-4, atol=1e-5)


def _close_reduction(got, ref, name):
    floor = 1e-5 + 1e-6 * float(np.abs(ref).max())
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=floor, err_msg=name)
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref), name


@pytest.mark.parametrize("n", [20000, 1000, 200])
def test_tc_backward_64_vs_oracle(fc, oracle_mod, n):
    """Full tensor-core backward (d_features, d_theta, d_theta_b, d_locations) at 64->64."""
    from paper_1803_07289_b200 import _ops

    k = 8
    t, h = _layer(n, 64, 64, k, seed=25)
    df, dth, dtb, dl = _ops.conv_backward(t["up"], t["feat"], t["loc"], t["nbr"], t["csr"], t["th"], t["tb"], 1, n,
                                          need=(True, True, True, True), mode="split")
    rdf, rdth, rdtb, rdl = oracle_mod.conv_backward(h["up"], h["feat"], h["loc"], h["nbr"], h["th"], h["tb"])
    np.testing.assert_allclose(df.cpu().numpy(), rdf, rtol=1e-4, atol=1e-5)
    _close_reduction(dth.cpu().numpy(), rdth, "d_theta")
    _close_reduction(dtb.cpu().numpy(), rdtb, "d_theta_b")
    _close_reduction(dl.cpu().numpy(), rdl, "d_locations")


def test_tc_backward_bitwise_deterministic(fc):
    import torch

    from paper_1803_07289_b200 import _ops

    n = 50000
    t, _ = _layer(n, 64, 64, 8, seed=26)
    run = lambda: _ops.conv_backward(t["up"], t["feat"], t["loc"], t["nbr"], t["csr"], t["th"], t["tb"], 1, n)  # noqa: E731
    a, b = run(), run()
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_tc_partial_tile_and_batch(fc, oracle_mod):
    """B=3 clouds of 1000 points (tiles straddle clouds, last tile partial)."""
    import torch

    from paper_1803_07289_b200 import _ops
    from paper_1803_07289_b200.core import synthetic_layer

    B, n, k, c = 3, 1000, 8, 64
    parts = [synthetic_layer(30 + b, 0, n, 3, c, c) for b in range(B)]
    dev = torch.device("cuda")
    loc = torch.from_numpy(np.concatenate([p[0] for p in parts])).to(dev, torch.float32)
    feat = torch.from_numpy(np.concatenate([p[1] for p in parts])).to(dev, torch.float32)
    th = torch.from_numpy(parts[0][2]).to(dev, torch.float32)
    tb = torch.from_numpy(parts[0][3]).to(dev, torch.float32)
    nbr = _ops.knn(loc, B, n, k)
    out = _ops.conv_forward(feat, loc, nbr, th, tb, B, n, "split").cpu().numpy()
    nb = nbr.cpu().numpy().astype(np.int64)
    for b in range(B):
        ref = oracle_mod.conv_forward(parts[b][1], parts[b][0], nb[b * n:(b + 1) * n], parts[0][2], parts[0][3])
        np.testing.assert_allclose(out[b * n:(b + 1) * n], ref, rtol=1e-4, atol=1e-5)


def test_tc_forward_deterministic_and_matches_simt_at_1M(fc):
    import torch

    from paper_1803_07289_b200 import _ops

    n, k = 1 << 20, 8
    t, _ = _layer(n, 64, 64, k, seed=23)
    a = _ops.conv_forward(t["feat"], t["loc"], t["nbr"], t["th"], t["tb"], 1, n, "split")
    b = _ops.conv_forward(t["feat"], t["loc"], t["nbr"], t["th"], t["tb"], 1, n, "split")
    assert torch.equal(a, b)
    s = _ops.conv_forward(t["feat"], t["loc"], t["nbr"], t["th"], t["tb"], 1, n, "simt")
    torch.testing.assert_close(a, s, rtol=1e-4, atol=1e-5)


def test_tc_adjoint_identity_at_1M(fc):
    """<A f, x> == <f, A^T x> for the split engine on a 1M-point cloud (fp64 dot products)."""
    from paper_1803_07289_b200 import _ops

    n, k = 1 << 20, 8
    t, _ = _layer(n, 64, 64, k, seed=24)
    af = _ops.conv_forward(t["feat"], t["loc"], t["nbr"], t["th"], t["tb"], 1, n, "split").double()
    atx = _ops.deconv_forward(t["up"], t["loc"], t["csr"], t["th"], t["tb"], 1, n, k, "split").double()
    lhs = float((af * t["up"].double()).sum())
    rhs = float((t["feat"].double() * atx).sum())
    scale = float(af.abs().sum() * t["up"].double().abs().max())
    assert abs(lhs - rhs) <= 1e-6 * scale, (lhs, rhs, scale)


@pytest.mark.parametrize("hub_degree", [40, 900])
def test_tc_reverse_long_lists_vs_oracle(fc, oracle_mod, hub_degree):
    """Reverse lists longer than the staged per-row limit (16) and 64-row groups whose lists
    overflow the stage capacity take the direct CSR path of the fast reverse kernel: a
    hand-built neighbourhood where `hub_degree` points all list a few hub points."""
    import torch

    from paper_1803_07289_b200 import _ops
    from paper_1803_07289_b200.core import synthetic_layer

    n, k = 4096, 8
    loc, feat, th, tb, up = synthetic_layer(41, 0, n, 3, 64, 64)
    rng = np.random.default_rng(7)
    nbr = np.empty((n, k), np.int64)
    nbr[:, 0] = np.arange(n)
    nbr[:, 1:] = rng.integers(0, n, size=(n, k - 1))
    hubs = [5, 70, 200]  # rows in different 64-row groups
    for h in hubs:
        rows = rng.choice(n, size=hub_degree, replace=False)
        nbr[rows, 1 + (h % (k - 1))] = h
    dev = torch.device("cuda")
    tl = {name: torch.from_numpy(v).to(dev, torch.float32) for name, v in
          dict(loc=loc, feat=feat, th=th, tb=tb, up=up).items()}
    nb = torch.from_numpy(nbr).to(dev, torch.int32)
    csr = _ops.csr_build(nb, 1, n)
    y = _ops.deconv_forward(tl["up"], tl["loc"], csr, tl["th"], tl["tb"], 1, n, k, "split").cpu().numpy()
    ref = oracle_mod.deconv_forward(up, loc, nbr, th, tb)
    np.testing.assert_allclose(y, ref, rtol=1e-4, atol=1e-5)
    df, _, _, dl = _ops.conv_backward(tl["up"], tl["feat"], tl["loc"], nb, csr, tl["th"], tl["tb"], 1, n,
                                      need=(True, True, True, True), mode="split")
    rdf, _, _, rdl = oracle_mod.conv_backward(up, feat, loc, nbr, th, tb)
    np.testing.assert_allclose(df.cpu().numpy(), rdf, rtol=1e-4, atol=1e-5)
    _close_reduction(dl.cpu().numpy(), rdl, "d_locations")


def test_tc_backward_batched_partial_tiles(fc, oracle_mod):
    """Warp-specialised backward kernels on B = 3 clouds of 1000 points (cloud-local
    neighbour indices, tiles straddling clouds, a partial last tile) vs the per-cloud oracle."""
    import torch

    from paper_1803_07289_b200 import _ops
    from paper_1803_07289_b200.core import synthetic_layer

    B, n, k, c = 3, 1000, 8, 64
    parts = [synthetic_layer(50 + b, 0, n, 3, c, c) for b in range(B)]
    dev = torch.device("cuda")
    cat = lambda i: torch.from_numpy(np.concatenate([p[i] for p in parts])).to(dev, torch.float32)  # noqa: E731
    loc, feat, up = cat(0), cat(1), cat(4)
    th = torch.from_numpy(parts[0][2]).to(dev, torch.float32)
    tb = torch.from_numpy(parts[0][3]).to(dev, torch.float32)
    nbr = _ops.knn(loc, B, n, k)
    csr = _ops.csr_build(nbr, B, n)
    df, dth, dtb, dl = _ops.conv_backward(up, feat, loc, nbr, csr, th, tb, B, n, need=(True, True, True, True),
                                          mode="split")
    nb = nbr.cpu().numpy().astype(np.int64)
    rdth = np.zeros_like(parts[0][2], dtype=np.float64)
    rdtb = np.zeros_like(parts[0][3], dtype=np.float64)
    for b in range(B):
        sl = slice(b * n, (b + 1) * n)
        rdf, r_th, r_tb, rdl = oracle_mod.conv_backward(parts[b][4], parts[b][1], parts[b][0], nb[sl], parts[0][2],
                                                        parts[0][3])
        np.testing.assert_allclose(df[sl].cpu().numpy(), rdf, rtol=1e-4, atol=1e-5)
        _close_reduction(dl[sl].cpu().numpy(), rdl, "d_locations")
        rdth += r_th
        rdtb += r_tb
    _close_reduction(dth.cpu().numpy(), rdth, "d_theta")
    _close_reduction(dtb.cpu().numpy(), rdtb, "d_theta_b")


def test_forward_rows_subset_equals_full_forward():
    """fc_conv_forward_rows (a shard's interior rows while the halo is in flight, then its
    boundary rows): every listed row bitwise equal to the full forward, other rows untouched."""
    import torch

    from paper_1803_07289_b200 import _ops

    n, k = 50_000, 8
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    pos = (torch.floor(torch.rand(n, 3, device="cuda", dtype=torch.float64, generator=g) * 2 ** 24) / 2 ** 24).float()
    pos = pos[_ops.spatial_order(pos).long()].contiguous()
    nbr = _ops.knn(pos, 1, n, k)
    feat = torch.randn(n, 64, device="cuda", generator=g)
    th = 0.1 * torch.randn(64, 64, 3, device="cuda", generator=g)
    tb = 0.1 * torch.randn(64, 64, device="cuda", generator=g)
    full = _ops.conv_forward(feat, pos, nbr, th, tb, 1, n)
    pick = torch.rand(n, device="cuda", generator=g) < 0.7
    a = torch.nonzero(pick).flatten().int()
    b = torch.nonzero(~pick).flatten().int()
    out = torch.full((n, 64), float("nan"), device="cuda")
    _ops.conv_forward_rows(feat, pos, nbr, th, tb, a, out)
    assert torch.isnan(out[b.long()]).all()
    assert torch.equal(out[a.long()], full[a.long()])
    _ops.conv_forward_rows(feat, pos, nbr, th, tb, b, out)
    assert torch.equal(out, full)
    out.fill_(float("nan"))
    _ops.conv_forward_rows(feat, pos, nbr, th, tb, a[:0], out)  # empty list: no work
    assert torch.isnan(out).all()

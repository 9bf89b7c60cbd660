"""GPU: point-chunk sharding with halos, emulated in one process (LocalTransport) with the
CUDA engines as the per-shard compute, against the unsharded CUDA operator; and batch
sharding of the torch ops."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_emulated_point_chunk_sharding_matches_unsharded(fc):
    import torch

    from paper_1803_07289_b200 import _ops, parallel
    from paper_1803_07289_b200.core import synthetic_layer

    n, k, c, world = 200_000, 8, 64, 4
    loc, feat, th, tb, up = synthetic_layer(51, 0, n, 3, c, c)
    dev = torch.device("cuda")
    pos = torch.from_numpy(loc).to(dev, torch.float32)
    order = _ops.spatial_order(pos).long()
    pos = pos[order].contiguous()
    f = torch.from_numpy(feat).to(dev, torch.float32)[order].contiguous()
    g = torch.from_numpy(up).to(dev, torch.float32)[order].contiguous()
    theta = torch.from_numpy(th).to(dev, torch.float32)
    theta_b = torch.from_numpy(tb).to(dev, torch.float32)
    nbr = _ops.knn(pos, 1, n, k)
    csr = _ops.csr_build(nbr, 1, n)
    ref_out = _ops.conv_forward(f, pos, nbr, theta, theta_b, 1, n)
    rdf, rdth, rdtb, rdl = _ops.conv_backward(g, f, pos, nbr, csr, theta, theta_b, 1, n)

    plans = parallel.HaloPlan.build_all(nbr.cpu().numpy(), world)
    tr = parallel.LocalTransport(world)
    for p in plans:
        p.post_halo(f[p.lo:p.hi], tr)
    feat_l = [p.gather_halo(f[p.lo:p.hi], tr) for p in plans]
    for p in plans:
        p.post_halo(pos[p.lo:p.hi], tr)
    loc_l = [p.gather_halo(pos[p.lo:p.hi], tr) for p in plans]
    outs = [parallel.sharded_forward(p, feat_l[r], loc_l[r], theta, theta_b) for r, p in enumerate(plans)]
    # forward rows are computed from identical inputs in identical order: bitwise equal
    assert torch.equal(torch.cat(outs), ref_out)

    parts = [parallel.sharded_backward_local(p, g[p.lo:p.hi], feat_l[r], loc_l[r], theta, theta_b)
             for r, p in enumerate(plans)]
    for r, p in enumerate(plans):
        p.post_partials(parts[r][0], tr)
    df = torch.cat([p.scatter_halo_add(parts[r][0], tr) for r, p in enumerate(plans)])
    for r, p in enumerate(plans):
        p.post_partials(parts[r][3], tr)
    dl = torch.cat([p.scatter_halo_add(parts[r][3], tr) for r, p in enumerate(plans)])
    dth = sum(x[1].double() for x in parts).float()
    dtb = sum(x[2].double() for x in parts).float()
    torch.testing.assert_close(df, rdf, rtol=1e-4, atol=1e-5)
    for got, ref in ((dth, rdth), (dtb, rdtb), (dl, rdl)):
        ref = ref.double()
        err = (got.double() - ref).abs().max() / ref.abs().max()
        assert err < 1e-5, float(err)

"""Fused downsample / upsample pooling (fc_pool_select_forward / _backward) against the
unfused composition the reference performs (flexops.py:168-203, network.py:248-280):
  PoolDown  = pool every fine point, gather the selection; backward = scatter_to_fine +
              flex_max_pool_backward over the full record
  Upsample  = scatter_to_fine (zero fill) + pool; backward = pool backward + gather
Bitwise equal (same comparisons, same additions), fp64 and fp32, with odd channel counts
(scalar path) and 16-byte-aligned ones (vector path); plus the oracle for the values."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cloud(n, k, c, dtype, seed):
    from paper_1803_07289_b200 import _ops

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    pos = (torch.floor(torch.rand(n, 3, generator=g, device="cuda", dtype=torch.float64) * 2 ** 10) / 2 ** 10)
    feat = torch.randn(n, c, generator=g, device="cuda", dtype=torch.float64)
    feat = torch.where(feat.abs() < 0.3, torch.zeros_like(feat), feat).to(dtype)  # ties, zeros
    nbr = _ops.knn(pos.float(), 1, n, k)
    csr = _ops.csr_build(nbr, 1, n)
    sel = torch.randperm(n, generator=torch.Generator().manual_seed(seed))[: n // 4].to(torch.int32).cuda()
    return pos, feat, nbr, csr, sel


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("c", [8, 13, 64])
def test_pool_down_fused_equals_composition(fc, dtype, c):
    from paper_1803_07289_b200 import _ops

    n, k = 1500, 9
    pos, feat, nbr, csr, sel = _cloud(n, k, c, dtype, 3 + c)
    m = sel.numel()
    pooled, am = _ops.pool_forward(feat, nbr, 1, n)
    ref_y = _ops.gather_rows(pooled, sel)
    y, win = _ops.pool_select_forward(feat, nbr, m, rows=sel)
    assert torch.equal(y, ref_y) and torch.equal(win, am[sel.long()])
    g = torch.randn(m, c, device="cuda", dtype=torch.float64).to(dtype)
    ref_d = _ops.pool_backward(_ops.scatter_rows(g, sel, n), am, csr, 1, n, k)
    d = _ops.pool_select_backward(g, win, csr, n, n, k, owner=_ops.selection_owner(sel, n))
    assert torch.equal(d, ref_d)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("c", [8, 13, 64])
def test_upsample_fused_equals_composition(fc, dtype, c):
    from paper_1803_07289_b200 import _ops

    n, k = 1500, 9
    pos, _, nbr, csr, sel = _cloud(n, k, c, dtype, 7 + c)
    m = sel.numel()
    coarse = torch.randn(m, c, device="cuda", dtype=torch.float64).to(dtype)
    full = _ops.scatter_rows(coarse, sel, n)
    ref_y, ref_am = _ops.pool_forward(full, nbr, 1, n)
    y, win = _ops.pool_select_forward(coarse, nbr, n, owner=_ops.selection_owner(sel, n))
    assert torch.equal(y, ref_y) and torch.equal(win, ref_am)
    g = torch.randn(n, c, device="cuda", dtype=torch.float64).to(dtype)
    ref_d = _ops.gather_rows(_ops.pool_backward(g, ref_am, csr, 1, n, k), sel)
    d = _ops.pool_select_backward(g, win, csr, m, n, k, rows=sel)
    assert torch.equal(d, ref_d)


def test_flex_upsample_matches_oracle(fc, oracle_mod):
    """numpy API (fp64): the fused flex_upsample equals the reference's scatter + pool."""
    rng = np.random.default_rng(1)
    n, k, c = 800, 7, 5
    loc = np.floor(rng.random((n, 3)) * 2 ** 10) / 2 ** 10
    nbr = oracle_mod.knn_brute(loc, k)
    sel = rng.permutation(n)[:200]
    coarse = rng.standard_normal((200, c))
    full = np.zeros((n, c))
    full[sel] = coarse
    ref_p, ref_a = oracle_mod.pool_forward(full, nbr)
    pooled, record = fc.flex_upsample(coarse, sel, fc.NeighborIndex(nbr), n, with_record=True)
    np.testing.assert_array_equal(pooled, ref_p)
    np.testing.assert_array_equal(record, ref_a)

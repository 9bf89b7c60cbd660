"""Batched torch operator surface of the north_star: flex_conv, flex_pool, flex_deconv
and the kNN neighbourhood builder on [B, D, N] features, [B, Dp, N] positions and
[B, K, N] int neighbourhoods, with the reference's theta [Dout, Din, Dp] / theta_b
[Dout, Din] shapes, differentiable through torch.autograd.

Storage is point-major ([B, N, D]: a neighbour's D channels are one contiguous row);
a [B, D, N] argument that is the transpose view of point-major storage (what these
ops return) is consumed without a copy, anything else is transposed once.  Offsets are
centre - neighbour, as in the reference (_native.pyx:55); the paper's neighbour-centre
form is the same operator with -theta.
"""

from __future__ import annotations

import torch

from . import _lib, _ops
from .errors import ShapeMismatchError


def _pm(x: torch.Tensor, name: str) -> torch.Tensor:
    """[B, D, N] -> point-major [B*N, D] (a view when x is a transposed point-major tensor)."""
    if x.dim() != 3:
        raise ShapeMismatchError(f"{name} must be [B, D, N], got {tuple(x.shape)}")
    b, d, n = x.shape
    pm = x.transpose(1, 2)
    if not pm.is_contiguous():
        pm = pm.contiguous()
    return pm.reshape(b * n, d)


def _bdn(pm: torch.Tensor, b: int, n: int) -> torch.Tensor:
    return pm.view(b, n, pm.shape[-1]).transpose(1, 2)


class Neighborhood:
    """A [B, K, N] neighbourhood (cloud-local indices) with its device int32 table and the
    cached reverse neighbourhood used by the backward passes and flex_deconv."""

    def __init__(self, table_bnk: torch.Tensor, validate: bool = True):
        if table_bnk.dim() != 3:
            raise ShapeMismatchError(f"neighbourhood storage must be [B, N, K], got {tuple(table_bnk.shape)}")
        if table_bnk.dtype != torch.int32:
            table_bnk = table_bnk.to(torch.int32)
        self.table = table_bnk.contiguous()
        self.batch, self.n, self.k = (int(s) for s in self.table.shape)
        if validate:
            bad = _ops.check_indices(self.table, self.n)
            if int(bad.item()):
                from .errors import IndexOutOfRangeError

                raise IndexOutOfRangeError("neighborhood index out of [0, N)")
        self._csr = None

    @classmethod
    def from_bkn(cls, nbr: torch.Tensor, validate: bool = True) -> "Neighborhood":
        """From the north_star [B, K, N] layout."""
        if isinstance(nbr, Neighborhood):
            return nbr
        if nbr.dim() != 3:
            raise ShapeMismatchError(f"neighborhood must be [B, K, N], got {tuple(nbr.shape)}")
        return cls(nbr.transpose(1, 2), validate=validate)

    @property
    def bkn(self) -> torch.Tensor:
        """[B, K, N] view (no copy)."""
        return self.table.transpose(1, 2)

    @property
    def flat(self) -> torch.Tensor:
        return self.table.view(self.batch * self.n, self.k)

    def csr(self):
        """Reverse neighbourhood, built on first use on the current stream without a host
        sync (the table was range-checked when this Neighborhood was created, or came from
        knn), so a backward that first needs it stays CUDA-graph capturable."""
        if self._csr is None:
            self._csr = _ops.csr_build(self.flat, self.batch, self.n, validate=False)
        return self._csr


def knn(positions: torch.Tensor, k: int, algo: str = "auto") -> Neighborhood:
    """Exact self-kNN neighbourhood of every cloud in positions [B, Dp, N]: row i is
    [i, the k-1 nearest others by (d^2, index)] (neighborhood.py:1-8, :149-187).
    Returns a Neighborhood; `.bkn` is the [B, K, N] int32 view."""
    b, dp, n = positions.shape
    pts = _pm(positions, "positions")
    a = {"auto": _lib.KNN_AUTO, "brute": _lib.KNN_BRUTE, "grid": _lib.KNN_GRID}[algo]
    table = _ops.knn(pts, b, n, int(k), a)
    return Neighborhood(table.view(b, n, k), validate=False)


def spatial_order(positions: torch.Tensor) -> torch.Tensor:
    """Cell-ordered permutation of one cloud [Dp, N] or [N, Dp] (returns int64 [N])."""
    pts = positions.t() if positions.shape[0] < positions.shape[1] else positions
    return _ops.spatial_order(pts.contiguous()).to(torch.int64)


class _FlexConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, feat, loc, theta, theta_b, nb: Neighborhood, mode):
        out = _ops.conv_forward(feat, loc, nb.flat, theta, theta_b, nb.batch, nb.n, mode)
        ctx.save_for_backward(feat, loc, theta, theta_b)
        ctx.nb, ctx.mode = nb, mode
        return out

    @staticmethod
    def backward(ctx, g):
        feat, loc, theta, theta_b = ctx.saved_tensors
        nb = ctx.nb
        need = (ctx.needs_input_grad[0], ctx.needs_input_grad[2], ctx.needs_input_grad[3], ctx.needs_input_grad[1])
        csr = nb.csr() if (need[0] or need[3]) else None
        df, dth, dtb, dl = _ops.conv_backward(g.contiguous(), feat, loc, nb.flat, csr, theta, theta_b, nb.batch,
                                              nb.n, need=need, mode=ctx.mode)
        return df, dl, dth, dtb, None, None


class _FlexDeconvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, loc, theta, theta_b, nb: Neighborhood, mode):
        y = _ops.deconv_forward(x, loc, nb.csr(), theta, theta_b, nb.batch, nb.n, nb.k, mode)
        ctx.save_for_backward(x, loc, theta, theta_b)
        ctx.nb, ctx.mode = nb, mode
        return y

    @staticmethod
    def backward(ctx, gy):
        # <A^T x, gy> = <x, A gy>: d_x = flex_conv(gy); theta/loc grads are flex_conv's
        # backward with upstream = x and features = gy.
        x, loc, theta, theta_b = ctx.saved_tensors
        nb = ctx.nb
        gy = gy.contiguous()
        dx = _ops.conv_forward(gy, loc, nb.flat, theta, theta_b, nb.batch, nb.n, ctx.mode) \
            if ctx.needs_input_grad[0] else None
        need_dl = ctx.needs_input_grad[1]
        dth = dtb = dl = None
        if ctx.needs_input_grad[2] or ctx.needs_input_grad[3] or need_dl:
            _, dth, dtb, dl = _ops.conv_backward(x, gy, loc, nb.flat, nb.csr() if need_dl else None, theta,
                                                 theta_b, nb.batch, nb.n,
                                                 need=(False, ctx.needs_input_grad[2], ctx.needs_input_grad[3],
                                                       need_dl), mode=ctx.mode)
        return dx, dl, dth, dtb, None, None


class _FlexPoolFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, feat, nb: Neighborhood):
        out, am = _ops.pool_forward(feat, nb.flat, nb.batch, nb.n)
        ctx.save_for_backward(am)
        ctx.nb = nb
        ctx.mark_non_differentiable(am)
        return out, am

    @staticmethod
    def backward(ctx, g, _g_am):
        (am,) = ctx.saved_tensors
        nb = ctx.nb
        return _ops.pool_backward(g.contiguous(), am, nb.csr(), nb.batch, nb.n, nb.k), None


def _nbh(neighborhood) -> Neighborhood:
    return neighborhood if isinstance(neighborhood, Neighborhood) else Neighborhood.from_bkn(neighborhood)


def flex_conv(features, positions, neighborhood, theta, theta_b, mode: str = "auto"):
    """out[b, :, i] = sum_{j in N(i)} sum_c (<theta[:, c], p_i - p_j> + theta_b[:, c]) f[b, c, j].
    features [B, Din, N], positions [B, Dp, N], neighborhood [B, K, N] (or Neighborhood),
    theta [Dout, Din, Dp], theta_b [Dout, Din] -> [B, Dout, N]."""
    nb = _nbh(neighborhood)
    feat = _pm(features, "features")
    loc = _pm(positions, "positions")
    if feat.shape[0] != nb.batch * nb.n or loc.shape[0] != nb.batch * nb.n:
        raise ShapeMismatchError("features / positions / neighborhood disagree on B*N")
    out = _FlexConvFn.apply(feat, loc, theta, theta_b, nb, mode)
    return _bdn(out, nb.batch, nb.n)


def flex_deconv(features, positions, neighborhood, theta, theta_b, mode: str = "auto"):
    """Transposed flex-convolution: the adjoint of flex_conv with the same theta/theta_b
    ([Dout, Din, Dp] / [Dout, Din]).  features [B, Dout, N] -> [B, Din, N]."""
    nb = _nbh(neighborhood)
    x = _pm(features, "features")
    loc = _pm(positions, "positions")
    y = _FlexDeconvFn.apply(x, loc, theta, theta_b, nb, mode)
    return _bdn(y, nb.batch, nb.n)


def flex_pool(features, neighborhood, return_argmax: bool = False):
    """Neighbourhood max-pool: out[b, c, i] = max_{j in N(i)} f[b, c, j]; ties to the lowest
    index (_native.pyx:151).  Optional argmax [B, D, N] int32 (cloud-local winner)."""
    nb = _nbh(neighborhood)
    feat = _pm(features, "features")
    out, am = _FlexPoolFn.apply(feat, nb)
    out = _bdn(out, nb.batch, nb.n)
    return (out, _bdn(am, nb.batch, nb.n)) if return_argmax else out

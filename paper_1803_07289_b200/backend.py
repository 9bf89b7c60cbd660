"""The reference's kernel-module ABI, implemented on the B200 library.

The reference selects its kernel module through backend.active() and calls it with
numpy float64 / int64 buffers and caller-allocated outputs (backend.py:34-62;
signatures _native.pyx:25-28, 69-74, 130-132, 158-159, 171-176 and _reference.py).
This module exposes the same five entry points with the same signatures and in-place
output contract, so it can be installed in the reference's backend slot unchanged
(INTEGRATION.md):  `flexconv.backend._active = paper_1803_07289_b200.backend`.
Arithmetic: the fp64 engine (reference operation order, bitwise-identical forward and
pooling); `num_threads` is accepted and ignored.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib, _ops

KERNEL_VERSION = 1


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _t(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(_dev(), dtype=dtype)


def _nbr(neighbors, n):
    t = _t(neighbors, torch.int64)
    table, _ = _ops.narrow_indices(t, n)
    return table


def flex_conv_forward(features, locations, neighbors, theta, theta_b, out, num_threads):
    n = features.shape[0]
    res = _ops.conv_forward(_t(features), _t(locations), _nbr(neighbors, n), _t(theta), _t(theta_b), 1, n)
    out[...] = res.cpu().numpy()
    return out


def flex_conv_backward(upstream, features, locations, neighbors, theta, theta_b,
                       d_features, d_locations, d_theta, d_theta_b, with_locations):
    """Accumulates into the caller's (zero-filled) outputs, as the reference kernel does."""
    n = features.shape[0]
    table = _nbr(neighbors, n)
    csr = _ops.csr_build(table, 1, n)
    df, dth, dtb, dl = _ops.conv_backward(_t(upstream), _t(features), _t(locations), table, csr, _t(theta),
                                          _t(theta_b), 1, n, need=(True, True, True, bool(with_locations)))
    d_features += df.cpu().numpy()
    d_theta += dth.cpu().numpy()
    d_theta_b += dtb.cpu().numpy()
    if with_locations:
        d_locations += dl.cpu().numpy()
    return d_features


def max_pool_forward(features, neighbors, out, argmax, num_threads):
    n = neighbors.shape[0]
    o, am = _ops.pool_forward(_t(features), _nbr(neighbors, features.shape[0]), 1, n)
    out[...] = o.cpu().numpy()
    argmax[...] = am.to(torch.int64).cpu().numpy()
    return out


def max_pool_backward(upstream, argmax, d_features):
    rows = d_features.shape[0]
    rec, _ = _ops.narrow_indices(_t(argmax, torch.int64), rows)
    d_features += _ops.pool_backward_record(_t(upstream), rec, rows).cpu().numpy()
    return d_features


def knn_self_query(points, axis, split, left, right, lo, hi, perm, k, out, num_threads):
    """The kd-tree arrays are ignored: the GPU kNN needs only the points."""
    n = points.shape[0]
    res = _ops.knn(_t(points), 1, n, int(k), _lib.KNN_AUTO)
    out[...] = res.to(torch.int64).cpu().numpy()
    return out

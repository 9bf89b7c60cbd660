"""The reference's operator API (/root/reference/pkg/src/flexconv/flexops.py) on the
B200 kernels: same names, arguments, shapes, return types and exceptions.

Inputs may be numpy arrays (the reference's types) or torch tensors:
  * numpy in -> numpy out, computed in fp64 on the GPU (the reference coerces every
    float to float64, flexops.py:30-31,70-74); the fp64 engine follows the reference's
    operation order, so forward and pooling results are bitwise identical to _native.
  * torch in -> torch out on the same device, computed in the tensor's dtype
    (float32 selects the fp32 engines: `mode` = "auto" | "simt" | "split" | "bf16").
There is no CPU implementation: the arithmetic always runs in libflexconv_b200.so.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _ops
from .errors import IndexOutOfRangeError, NonFiniteError, ShapeMismatchError
from .neighborhood import NeighborIndex


def _device():
    return torch.device("cuda", torch.cuda.current_device())


class _Kind:
    """Remembers whether the caller passed numpy (-> return numpy) or torch."""

    def __init__(self, *arrays):
        self.numpy = not any(isinstance(a, torch.Tensor) for a in arrays)
        dev = next((a.device for a in arrays if isinstance(a, torch.Tensor)), None)
        self.out_device = dev
        self.device = dev if (dev is not None and dev.type == "cuda") else _device()
        ft = next((a.dtype for a in arrays if isinstance(a, torch.Tensor) and a.is_floating_point()), None)
        self.dtype = torch.float64 if (self.numpy or ft is None) else ft

    def dev(self, a, dtype=None):
        dtype = dtype or self.dtype
        t = torch.from_numpy(np.ascontiguousarray(a)) if not isinstance(a, torch.Tensor) else a
        return t.to(device=self.device, dtype=dtype).contiguous()

    def back(self, t):
        if t is None:
            return None
        if self.numpy:
            return t.cpu().numpy()
        return t if self.out_device is None else t.to(self.out_device)


def _f64_2d(a, name):
    if isinstance(a, torch.Tensor):
        if a.dim() != 2:
            raise ShapeMismatchError(f"{name} must be 2-d, got shape {tuple(a.shape)}")
        return a
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ShapeMismatchError(f"{name} must be 2-d, got shape {a.shape}")
    return a


@dataclass
class FlexConvParams:
    """theta: C_out x C_in x d offset weights; theta_b: C_out x C_in biases (flexops.py:22-51)."""

    theta: object
    theta_b: object

    def __post_init__(self):
        if isinstance(self.theta, torch.Tensor) or isinstance(self.theta_b, torch.Tensor):
            self.theta = torch.as_tensor(self.theta)
            self.theta_b = torch.as_tensor(self.theta_b)
            finite = bool(torch.isfinite(self.theta).all()) and bool(torch.isfinite(self.theta_b).all())
        else:
            self.theta = np.ascontiguousarray(self.theta, dtype=np.float64)
            self.theta_b = np.ascontiguousarray(self.theta_b, dtype=np.float64)
            finite = bool(np.isfinite(self.theta).all() and np.isfinite(self.theta_b).all())
        if self.theta.ndim != 3 or self.theta_b.ndim != 2:
            raise ShapeMismatchError("theta must be C_out x C_in x d, theta_b C_out x C_in")
        if tuple(self.theta.shape[:2]) != tuple(self.theta_b.shape):
            raise ShapeMismatchError(
                f"theta {tuple(self.theta.shape)} and theta_b {tuple(self.theta_b.shape)} disagree")
        if not finite:
            raise NonFiniteError("parameters contain NaN or Inf")

    @classmethod
    def _checked_views(cls, theta: torch.Tensor, theta_b: torch.Tensor) -> "FlexConvParams":
        """Views into a parameter vector whose finiteness the caller has already checked
        once for the whole vector (network.LayerGraph.forward): the shape checks of
        __post_init__ without a per-layer device->host sync."""
        self = cls.__new__(cls)
        self.theta, self.theta_b = theta, theta_b
        if theta.ndim != 3 or theta_b.ndim != 2 or tuple(theta.shape[:2]) != tuple(theta_b.shape):
            raise ShapeMismatchError("theta must be C_out x C_in x d, theta_b C_out x C_in")
        return self

    @property
    def c_out(self) -> int:
        return int(self.theta.shape[0])

    @property
    def c_in(self) -> int:
        return int(self.theta.shape[1])

    @property
    def d(self) -> int:
        return int(self.theta.shape[2])


@dataclass
class GradBundle:
    """Gradients mirroring the forward arguments (flexops.py:54-61)."""

    d_features: object
    d_theta: object
    d_theta_b: object
    d_locations: object | None


def param_count(c_in: int, c_out: int, d: int) -> int:
    """C_out*C_in*(d+1) trainable scalars per layer (flexops.py:64-67)."""
    return c_out * c_in * (d + 1)


def _check_conv_args(features, locations, neighbors: NeighborIndex, params: FlexConvParams):
    """flexops.py:77-94: shapes, then the index range (checked once per device)."""
    features = _f64_2d(features, "features")
    locations = _f64_2d(locations, "locations")
    n = int(features.shape[0])
    if int(locations.shape[0]) != n:
        raise ShapeMismatchError(f"{n} feature rows but {locations.shape[0]} locations")
    if params.c_in != int(features.shape[1]):
        raise ShapeMismatchError(f"params expect C={params.c_in}, features have C={features.shape[1]}")
    if params.d != int(locations.shape[1]):
        raise ShapeMismatchError(f"params expect d={params.d}, locations have d={locations.shape[1]}")
    if neighbors.n != n:
        raise ShapeMismatchError(f"neighbor index has {neighbors.n} rows for {n} points")
    return features, locations


def flex_conv_forward(features, locations, neighbors: NeighborIndex, params: FlexConvParams,
                      num_threads: int = 1, *, mode: str = "auto"):
    """f'(i, c') = sum_c sum_{j in N(i)} (<theta[c',c], l_i - l_j> + theta_b[c',c]) f(j, c)
    (flexops.py:97-110).  `num_threads` is accepted and ignored."""
    features, locations = _check_conv_args(features, locations, neighbors, params)
    kd = _Kind(features, locations, params.theta)
    n = int(features.shape[0])
    table = neighbors.device_table(kd.device, n)
    out = _ops.conv_forward(kd.dev(features), kd.dev(locations), table, kd.dev(params.theta),
                            kd.dev(params.theta_b), 1, n, mode)
    return kd.back(out)


def flex_conv_backward(upstream, features, locations, neighbors: NeighborIndex, params: FlexConvParams,
                       with_locations: bool = True, *, mode: str = "auto") -> GradBundle:
    """Exact analytic gradients w.r.t. features, theta, theta_b and both location roles
    (flexops.py:113-132).  Deterministic: bitwise reproducible run to run."""
    features, locations = _check_conv_args(features, locations, neighbors, params)
    upstream = _f64_2d(upstream, "upstream")
    n = int(features.shape[0])
    if tuple(upstream.shape) != (n, params.c_out):
        raise ShapeMismatchError(f"upstream must be {(n, params.c_out)}, got {tuple(upstream.shape)}")
    kd = _Kind(features, locations, upstream, params.theta)
    table = neighbors.device_table(kd.device, n)
    csr = neighbors.reverse(kd.device, n)
    df, dth, dtb, dl = _ops.conv_backward(kd.dev(upstream), kd.dev(features), kd.dev(locations), table, csr,
                                          kd.dev(params.theta), kd.dev(params.theta_b), 1, n,
                                          need=(True, True, True, bool(with_locations)), mode=mode)
    return GradBundle(kd.back(df), kd.back(dth), kd.back(dtb), kd.back(dl) if with_locations else None)


def flex_deconv_forward(x, locations, neighbors: NeighborIndex, params: FlexConvParams, *, mode: str = "auto"):
    """Transposed flex-convolution y = A(theta)^T x (the adjoint of flex_conv_forward with
    the same params).  No reference function; equals the reference's
    flex_conv_backward(upstream=x, ...).d_features (_native.pyx:106-120)."""
    x = _f64_2d(x, "x")
    locations = _f64_2d(locations, "locations")
    n = int(x.shape[0])
    if int(x.shape[1]) != params.c_out:
        raise ShapeMismatchError(f"x must have C_out={params.c_out} channels, got {x.shape[1]}")
    if int(locations.shape[0]) != n or neighbors.n != n:
        raise ShapeMismatchError("x, locations and neighbors disagree on n")
    if params.d != int(locations.shape[1]):
        raise ShapeMismatchError(f"params expect d={params.d}, locations have d={locations.shape[1]}")
    kd = _Kind(x, locations, params.theta)
    csr = neighbors.reverse(kd.device, n)
    y = _ops.deconv_forward(kd.dev(x), kd.dev(locations), csr, kd.dev(params.theta), kd.dev(params.theta_b),
                            1, n, neighbors.k, mode)
    return kd.back(y)


def flex_max_pool(features, neighbors: NeighborIndex, num_threads: int = 1):
    """Per-point, per-channel max over the neighbourhood; returns (pooled, argmax record),
    ties to the lowest global index (flexops.py:135-151).  The record is int64."""
    features = _f64_2d(features, "features")
    if neighbors.n != int(features.shape[0]):
        raise ShapeMismatchError(f"neighbor index has {neighbors.n} rows for {features.shape[0]} points")
    kd = _Kind(features)
    n = int(features.shape[0])
    table = neighbors.device_table(kd.device, n)
    out, am = _ops.pool_forward(kd.dev(features), table, 1, n)
    am = am.to(torch.int64)
    return kd.back(out), kd.back(am)


def flex_max_pool_backward(upstream, record, n: int | None = None):
    """Route each upstream entry to its recorded winner (flexops.py:154-165)."""
    upstream = _f64_2d(upstream, "upstream")
    kd = _Kind(upstream)
    rec = record if isinstance(record, torch.Tensor) else np.ascontiguousarray(record, dtype=np.int64)
    if tuple(rec.shape) != tuple(upstream.shape):
        raise ShapeMismatchError(f"record shape {tuple(rec.shape)} != upstream {tuple(upstream.shape)}")
    rows = int(upstream.shape[0]) if n is None else int(n)
    rec_t = kd.dev(rec, dtype=torch.int64)
    rec32, bad = _ops.narrow_indices(rec_t, rows)
    if rec_t.numel() and int(bad.item()):
        raise IndexOutOfRangeError("corrupt pool record: winner index out of range")
    df = _ops.pool_backward_record(kd.dev(upstream), rec32, rows)
    return kd.back(df)


def _selection(sel, kd: _Kind, hi: int):
    s = sel if isinstance(sel, torch.Tensor) else np.asarray(sel, dtype=np.int64)
    s_t = kd.dev(s, dtype=torch.int64).reshape(-1)
    s32, bad = _ops.narrow_indices(s_t, hi)
    if s_t.numel() and int(bad.item()):
        raise IndexOutOfRangeError("selection index out of [0, n)")
    return s32


def downsample_gather(features, selection):
    """Row-gather of the selected indices (flexops.py:168-175)."""
    features = _f64_2d(features, "features")
    kd = _Kind(features)
    s32 = _selection(selection, kd, int(features.shape[0]))
    return kd.back(_ops.gather_rows(kd.dev(features), s32))


def scatter_to_fine(features_coarse, selection, n: int):
    """Copy coarse rows to their fine positions, zero elsewhere (flexops.py:178-190)."""
    features_coarse = _f64_2d(features_coarse, "features_coarse")
    kd = _Kind(features_coarse)
    nsel = int(np.asarray(selection).shape[0]) if not isinstance(selection, torch.Tensor) else int(selection.shape[0])
    if nsel != int(features_coarse.shape[0]):
        raise ShapeMismatchError(f"{features_coarse.shape[0]} coarse rows but {nsel} selections")
    s32 = _selection(selection, kd, int(n))
    return kd.back(_ops.scatter_rows(kd.dev(features_coarse), s32, int(n)))


def flex_upsample(features_coarse, selection, fine_neighbors: NeighborIndex, n: int,
                  num_threads: int = 1, with_record: bool = False):
    """Scatter coarse features to the fine level (zero fill) and flex-max-pool there
    (flexops.py:193-203)."""
    features_coarse = _f64_2d(features_coarse, "features_coarse")
    kd = _Kind(features_coarse)
    nsel = int(np.asarray(selection).shape[0]) if not isinstance(selection, torch.Tensor) else int(selection.shape[0])
    if nsel != int(features_coarse.shape[0]):
        raise ShapeMismatchError(f"{features_coarse.shape[0]} coarse rows but {nsel} selections")
    if fine_neighbors.n != int(n):
        raise ShapeMismatchError(f"neighbor index has {fine_neighbors.n} rows for {n} points")
    s32 = _selection(selection, kd, int(n))
    table = fine_neighbors.device_table(kd.device, int(n))
    # fused scatter + pool (fc_pool_select_forward): no zero-filled fine-level intermediate
    pooled, record = _ops.pool_select_forward(kd.dev(features_coarse), table, int(n),
                                              owner=_ops.selection_owner(s32, int(n)))
    pooled, record = kd.back(pooled), kd.back(record.to(torch.int64))
    return (pooled, record) if with_record else pooled


def pointwise_conv(features, weights, bias):
    """Per-point affine map out = f @ W.T + b (flexops.py:206-217).  Not part of the
    flex-conv hot path: a plain GEMM, delegated to cuBLAS."""
    features = _f64_2d(features, "features")
    weights = _f64_2d(weights, "weights")
    if int(weights.shape[1]) != int(features.shape[1]):
        raise ShapeMismatchError(f"weights expect C={weights.shape[1]}, features have C={features.shape[1]}")
    kd = _Kind(features, weights, bias)
    b = kd.dev(bias).reshape(-1)
    if tuple(b.shape) != (int(weights.shape[0]),):
        raise ShapeMismatchError(f"bias must have shape ({weights.shape[0]},), got {tuple(b.shape)}")
    return kd.back(torch.addmm(b, kd.dev(features), kd.dev(weights).t()))


def pointwise_conv_backward(upstream, features, weights):
    """Matrix-calculus gradients of the per-point affine map (flexops.py:220-226)."""
    kd = _Kind(upstream, features, weights)
    g, f, w = kd.dev(upstream), kd.dev(features), kd.dev(weights)
    return kd.back(g @ w), kd.back(g.t() @ f), kd.back(g.sum(0))

"""Device-level operator layer: torch CUDA tensors in the point-major layout, one C-ABI
call per operator (include/flexconv_b200.h).  torch supplies allocation and the current
stream only; every byte of arithmetic runs in libflexconv_b200.so.

Shapes (T = B*N points, B clouds of N points stacked along the point axis):
  features [T, C], locations [T, d], neighbours [T, K] int32 (cloud-local indices),
  theta [C_out, C_in, d], theta_b [C_out, C_in], reverse CSR (offsets [T+1], entries [T*K]).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import ShapeMismatchError, UnsupportedError

MODES = {"auto": _lib.MODE_AUTO, "simt": _lib.MODE_SIMT, "split": _lib.MODE_TC_SPLIT,
         "bf16": _lib.MODE_TC_BF16}


def _mode(mode) -> int:
    if isinstance(mode, int):
        return mode
    try:
        return MODES[mode]
    except KeyError as exc:
        raise UnsupportedError(f"unknown engine {mode!r}; choose from {sorted(MODES)}") from exc


def _dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.FC_F32
    if t.dtype == torch.float64:
        return _lib.FC_F64
    raise UnsupportedError(f"floating tensors must be float32 or float64, got {t.dtype}")


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _call(dev: torch.device, name: str, *args) -> None:
    """One C-ABI call with `dev` as the current CUDA device: the library launches on the
    current device, and the stream passed in belongs to `dev` (a tensor on cuda:1 while
    cuda:0 is current would otherwise be launched into the wrong device's stream)."""
    if dev.index is None or dev.index == torch.cuda.current_device():
        _lib.call(name, *args)
    else:
        with torch.cuda.device(dev):
            _lib.call(name, *args)


def _shape(t: torch.Tensor, want: tuple, name: str) -> None:
    if tuple(t.shape) != tuple(want):
        raise ShapeMismatchError(f"{name} has shape {tuple(t.shape)}, expected {tuple(want)}")


def _conv_shapes(theta, theta_b):
    if theta.dim() != 3:
        raise ShapeMismatchError(f"theta must be [C_out, C_in, d], got {tuple(theta.shape)}")
    c_out, c_in, d = theta.shape
    _shape(theta_b, (c_out, c_in), "theta_b")
    return c_out, c_in, d


def _stream(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _need(t: torch.Tensor, name: str, dtype=None, device=None):
    if not t.is_cuda:
        raise UnsupportedError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if dtype is not None and t.dtype != dtype:
        raise ShapeMismatchError(f"{name} must be {dtype}, got {t.dtype}")
    if device is not None and t.device != device:
        raise ShapeMismatchError(f"{name} is on {t.device}, expected {device}")
    return t.contiguous()


def csr_build(nbr: torch.Tensor, batch: int, n: int, validate: bool = True):
    """Reverse neighbourhood (stable counting sort): offsets [B*N+1], entries [B*N*K].
    validate=True checks the indices and raises IndexOutOfRangeError (one host sync, like
    the reference's range check); validate=False is the stream-ordered, graph-capturable
    build for tables that are valid by construction or were checked already."""
    nbr = _need(nbr, "neighbors", torch.int32)
    k = nbr.shape[-1]
    _shape(nbr, (batch * n, k), "neighbors")
    off = torch.empty(batch * n + 1, dtype=torch.int32, device=nbr.device)
    ent = torch.empty(batch * n * k, dtype=torch.int32, device=nbr.device)
    if validate:
        _call(nbr.device, "fc_csr_build", batch, n, k, _p(nbr), _p(off), _p(ent), _stream(nbr))
    else:
        bad = torch.zeros(1, dtype=torch.int32, device=nbr.device)
        _call(nbr.device, "fc_csr_build_async", batch, n, k, _p(nbr), _p(off), _p(ent), _p(bad), _stream(nbr))
    return off, ent


def conv_forward(feat, loc, nbr, theta, theta_b, batch, n, mode="auto"):
    feat = _need(feat, "features")
    dt, dev = feat.dtype, feat.device
    loc = _need(loc, "locations", dt, dev)
    nbr = _need(nbr, "neighbors", torch.int32, dev)
    theta = _need(theta, "theta", dt, dev)
    theta_b = _need(theta_b, "theta_b", dt, dev)
    c_out, c_in, d = _conv_shapes(theta, theta_b)
    k = nbr.shape[-1]
    _shape(feat, (batch * n, c_in), "features")
    _shape(loc, (batch * n, d), "locations")
    _shape(nbr, (batch * n, k), "neighbors")
    out = torch.empty(batch * n, c_out, dtype=dt, device=dev)
    _call(feat.device, "fc_conv_forward", _dtype(feat), _mode(mode), batch, n, c_in, d, k, c_out, _p(feat), _p(loc),
              _p(nbr), _p(theta), _p(theta_b), _p(out), _stream(feat))
    return out


def deconv_backward(gy, x, loc, nbr, csr, theta, theta_b, batch, n, need=(True, True, True, True), mode="auto"):
    """Gradient of y = flex_deconv(x): (d_x, d_theta, d_theta_b, d_locations) for upstream gy
    (fc_deconv_backward); entries not in `need` are None."""
    gy = _need(gy, "upstream")
    dt, dev = gy.dtype, gy.device
    x = _need(x, "x", dt, dev)
    loc = _need(loc, "locations", dt, dev)
    nbr = _need(nbr, "neighbors", torch.int32, dev)
    theta = _need(theta, "theta", dt, dev)
    theta_b = _need(theta_b, "theta_b", dt, dev)
    c_out, c_in, d = _conv_shapes(theta, theta_b)
    k = nbr.shape[-1]
    _shape(gy, (batch * n, c_in), "upstream")
    _shape(x, (batch * n, c_out), "x")
    _shape(loc, (batch * n, d), "locations")
    _shape(nbr, (batch * n, k), "neighbors")
    want_dx, want_dth, want_dtb, want_dl = need
    dx = torch.empty(batch * n, c_out, dtype=dt, device=dev) if want_dx else None
    dl = torch.empty(batch * n, d, dtype=dt, device=dev) if want_dl else None
    dth = torch.empty(c_out, c_in, d, dtype=dt, device=dev) if want_dth else None
    dtb = torch.empty(c_out, c_in, dtype=dt, device=dev) if want_dtb else None
    off, ent = (csr if csr is not None else (None, None))
    _call(dev, "fc_deconv_backward", _dtype(gy), _mode(mode), batch, n, c_in, d, k, c_out, _p(gy), _p(x), _p(loc),
          _p(nbr), _p(off), _p(ent), _p(theta), _p(theta_b), _p(dx), _p(dl), _p(dth), _p(dtb), _stream(gy))
    return dx, dth, dtb, dl


def scratch_peak_bytes(reset: bool = False) -> int:
    """Peak device scratch (bytes) the library's entry points took on this thread since the
    last reset (fc_scratch_peak_bytes); reset=True starts a new measurement."""
    lib = _lib.lib()
    if reset:
        lib.fc_scratch_peak_reset()
        return 0
    return int(lib.fc_scratch_peak_bytes())


def conv_forward_rows_supported(c_in, d, k, c_out, dtype) -> bool:
    return dtype == torch.float32 and (c_in, d, k, c_out) == (64, 3, 8, 64)


def conv_forward_rows(feat, loc, nbr, theta, theta_b, rows, out):
    """Write rows `rows` (sorted int32 row ids) of the forward of one cloud into `out` [n, C_out]
    (fc_conv_forward_rows; other rows untouched).  Used to overlap a shard's interior rows with
    its halo exchange."""
    feat = _need(feat, "features", torch.float32)
    dev = feat.device
    loc = _need(loc, "locations", torch.float32, dev)
    nbr = _need(nbr, "neighbors", torch.int32, dev)
    rows = _need(rows, "rows", torch.int32, dev)
    c_out, c_in, d = _conv_shapes(theta, theta_b)
    n, k = nbr.shape
    _shape(feat, (n, c_in), "features")
    _shape(loc, (n, d), "locations")
    _shape(out, (n, c_out), "out")
    if not out.is_contiguous():
        raise ShapeMismatchError("out must be contiguous")
    _call(dev, "fc_conv_forward_rows", n, c_in, d, k, c_out, _p(feat), _p(loc), _p(nbr), _p(_need(theta, "theta")),
          _p(_need(theta_b, "theta_b")), _p(rows), rows.numel(), _p(out), _stream(feat))
    return out


def _out_ok(t, shape, dt, dev, name):
    if tuple(t.shape) != tuple(shape) or t.dtype != dt or t.device != dev or not t.is_contiguous():
        raise ShapeMismatchError(f"{name}: expected contiguous {dt} {tuple(shape)} on {dev}, got {t.dtype} "
                                 f"{tuple(t.shape)} on {t.device}")


def conv_backward(g, feat, loc, nbr, csr, theta, theta_b, batch, n, need=(True, True, True, True),
                  mode="auto", d_theta_out=None, d_theta_b_out=None):
    """Returns (d_features, d_theta, d_theta_b, d_locations); entries not in `need` are None.
    d_theta_out / d_theta_b_out: contiguous tensors to write the parameter gradients into
    (e.g. views of a flat gradient vector) instead of new ones."""
    feat = _need(feat, "features")
    dt, dev = feat.dtype, feat.device
    g = _need(g, "upstream", dt, dev)
    loc = _need(loc, "locations", dt, dev)
    nbr = _need(nbr, "neighbors", torch.int32, dev)
    theta = _need(theta, "theta", dt, dev)
    theta_b = _need(theta_b, "theta_b", dt, dev)
    c_out, c_in, d = _conv_shapes(theta, theta_b)
    k = nbr.shape[-1]
    _shape(g, (batch * n, c_out), "upstream")
    _shape(feat, (batch * n, c_in), "features")
    _shape(loc, (batch * n, d), "locations")
    _shape(nbr, (batch * n, k), "neighbors")
    if csr is not None:
        _shape(csr[0], (batch * n + 1,), "reverse offsets")
        _shape(csr[1], (batch * n * k,), "reverse entries")
    want_df, want_dth, want_dtb, want_dl = need
    df = torch.empty(batch * n, c_in, dtype=dt, device=dev) if want_df else None
    dl = torch.empty(batch * n, d, dtype=dt, device=dev) if want_dl else None
    dth = dtb = None
    if want_dth:
        dth = d_theta_out if d_theta_out is not None else torch.empty(c_out, c_in, d, dtype=dt, device=dev)
        _out_ok(dth, (c_out, c_in, d), dt, dev, "d_theta_out")
    if want_dtb:
        dtb = d_theta_b_out if d_theta_b_out is not None else torch.empty(c_out, c_in, dtype=dt, device=dev)
        _out_ok(dtb, (c_out, c_in), dt, dev, "d_theta_b_out")
    off, ent = csr if csr is not None else (None, None)
    _call(feat.device, "fc_conv_backward", _dtype(feat), _mode(mode), batch, n, c_in, d, k, c_out, _p(g), _p(feat),
              _p(loc), _p(nbr), _p(off), _p(ent), _p(theta), _p(theta_b), _p(df), _p(dl), _p(dth), _p(dtb),
              _stream(feat))
    return df, dth, dtb, dl


def deconv_forward(x, loc, csr, theta, theta_b, batch, n, k, mode="auto"):
    """y = A(theta)^T x: x [T, C_out] -> y [T, C_in]."""
    x = _need(x, "x")
    dt, dev = x.dtype, x.device
    loc = _need(loc, "locations", dt, dev)
    theta = _need(theta, "theta", dt, dev)
    theta_b = _need(theta_b, "theta_b", dt, dev)
    c_out, c_in, d = _conv_shapes(theta, theta_b)
    _shape(x, (batch * n, c_out), "x")
    _shape(loc, (batch * n, d), "locations")
    off, ent = csr
    _shape(off, (batch * n + 1,), "reverse offsets")
    _shape(ent, (batch * n * k,), "reverse entries")
    y = torch.empty(batch * n, c_in, dtype=dt, device=dev)
    _call(x.device, "fc_deconv_forward", _dtype(x), _mode(mode), batch, n, c_in, d, k, c_out, _p(x), _p(loc),
              _p(off), _p(ent), _p(theta), _p(theta_b), _p(y), _stream(x))
    return y


def pool_forward(feat, nbr, batch, n):
    feat = _need(feat, "features")
    nbr = _need(nbr, "neighbors", torch.int32, feat.device)
    c = feat.shape[-1]
    k = nbr.shape[-1]
    _shape(feat, (batch * n, c), "features")
    _shape(nbr, (batch * n, k), "neighbors")
    out = torch.empty_like(feat)
    am = torch.empty(feat.shape, dtype=torch.int32, device=feat.device)
    _call(feat.device, "fc_pool_forward", _dtype(feat), batch, n, c, k, _p(feat), _p(nbr), _p(out), _p(am),
              _stream(feat))
    return out, am


def pool_backward(g, argmax, csr, batch, n, k):
    g = _need(g, "upstream")
    argmax = _need(argmax, "argmax", torch.int32, g.device)
    c = g.shape[-1]
    _shape(g, (batch * n, c), "upstream")
    _shape(argmax, (batch * n, c), "argmax")
    df = torch.empty_like(g)
    off, ent = csr
    _shape(off, (batch * n + 1,), "reverse offsets")
    _shape(ent, (batch * n * k,), "reverse entries")
    _call(g.device, "fc_pool_backward", _dtype(g), batch, n, c, k, _p(g), _p(argmax), _p(off), _p(ent), _p(df),
              _stream(g))
    return df


def pool_backward_record(g, record, n_rows):
    g = _need(g, "upstream")
    record = _need(record, "record", torch.int32, g.device)
    n_up, c = g.shape
    off = torch.empty(n_rows * c + 1, dtype=torch.int32, device=g.device)
    ent = torch.empty(max(n_up * c, 1), dtype=torch.int32, device=g.device)
    _call(g.device, "fc_record_csr_build", n_up, n_rows, c, _p(record), _p(off), _p(ent), _stream(g))
    df = torch.empty(n_rows, c, dtype=g.dtype, device=g.device)
    _call(g.device, "fc_pool_backward_record", _dtype(g), n_up, n_rows, c, _p(g), _p(off), _p(ent), _p(df), _stream(g))
    return df


def knn(points, batch, n, k, algo=_lib.KNN_AUTO):
    points = _need(points, "points")
    d = points.shape[-1]
    out = torch.empty(batch * n, k, dtype=torch.int32, device=points.device)
    _call(points.device, "fc_knn", _dtype(points), batch, n, d, k, _p(points), _p(out), int(algo), _stream(points))
    return out


def spatial_order(points):
    points = _need(points, "points")
    n, d = points.shape
    order = torch.empty(n, dtype=torch.int32, device=points.device)
    _call(points.device, "fc_spatial_order", _dtype(points), n, d, _p(points), _p(order), _stream(points))
    return order


def inverse_density(points, nbr):
    """phi [n] fp64 of the IDISS sampler (fc_inverse_density)."""
    points = _need(points, "points", torch.float64)
    nbr = _need(nbr, "neighbors", torch.int32)
    n, d = points.shape
    phi = torch.empty(n, dtype=torch.float64, device=points.device)
    _call(points.device, "fc_inverse_density", n, d, nbr.shape[1], _p(points), _p(nbr), _p(phi), _stream(points))
    return phi


def gather_rows(x, sel):
    x = _need(x, "features")
    sel = _need(sel, "selection", torch.int32, x.device)
    out = torch.empty(sel.numel(), x.shape[1], dtype=x.dtype, device=x.device)
    _call(x.device, "fc_gather_rows", _dtype(x), sel.numel(), x.shape[1], _p(x), _p(sel), _p(out), _stream(x))
    return out


def scatter_rows(x, sel, rows_out):
    x = _need(x, "features")
    sel = _need(sel, "selection", torch.int32, x.device)
    out = torch.empty(rows_out, x.shape[1], dtype=x.dtype, device=x.device)
    _call(x.device, "fc_scatter_rows", _dtype(x), x.shape[0], rows_out, x.shape[1], _p(x), _p(sel), _p(out),
              _stream(x))
    return out


def selection_owner(sel, n):
    """owner [n] int32: owner[sel[r]] = r (largest r on duplicates), -1 elsewhere."""
    sel = _need(sel, "selection", torch.int32)
    owner = torch.empty(n, dtype=torch.int32, device=sel.device)
    _call(sel.device, "fc_selection_owner", sel.numel(), n, _p(sel), _p(owner), _stream(sel))
    return owner


def pool_select_forward(feat, nbr, m, rows=None, owner=None):
    """Fused PoolDown (rows = selection) / Upsample (owner = selection_owner) pooling: m output
    rows, winners = fine neighbour indices (fc_pool_select_forward)."""
    feat = _need(feat, "features")
    nbr = _need(nbr, "neighbors", torch.int32, feat.device)
    n, k = nbr.shape
    c = feat.shape[1]
    out = torch.empty(m, c, dtype=feat.dtype, device=feat.device)
    win = torch.empty(m, c, dtype=torch.int32, device=feat.device)
    _call(feat.device, "fc_pool_select_forward", _dtype(feat), m, n, c, k, _p(feat), _p(nbr), _p(rows), _p(owner), _p(out),
              _p(win), _stream(feat))
    return out, win


def pool_select_backward(g, winners, csr, m, n, k, rows=None, owner=None):
    """Backward of pool_select_forward: d_features for m fine rows (all n, or rows=selection)."""
    g = _need(g, "upstream")
    winners = _need(winners, "winners", torch.int32, g.device)
    off, ent = csr
    df = torch.empty(m, g.shape[1], dtype=g.dtype, device=g.device)
    _call(g.device, "fc_pool_select_backward", _dtype(g), m, n, g.shape[1], k, _p(g), _p(winners), _p(off), _p(ent),
              _p(rows), _p(owner), _p(df), _stream(g))
    return df


def narrow_indices(idx64, hi):
    """int64 -> int32 with the reference's [0, hi) range check; returns (idx32, bad_count)."""
    idx64 = _need(idx64, "indices", torch.int64)
    out = torch.empty(idx64.shape, dtype=torch.int32, device=idx64.device)
    bad = torch.zeros(1, dtype=torch.int32, device=idx64.device)
    _call(idx64.device, "fc_indices_to_i32", _p(idx64), _p(out), idx64.numel(), int(hi), _p(bad), _stream(idx64))
    return out, bad


def check_indices(idx32, hi):
    idx32 = _need(idx32, "indices", torch.int32)
    bad = torch.zeros(1, dtype=torch.int32, device=idx32.device)
    _call(idx32.device, "fc_check_indices", _p(idx32), idx32.numel(), int(hi), _p(bad), _stream(idx32))
    return bad


def count_nonfinite(x, bad=None):
    """Device int32 [1]: number of NaN / inf entries of x (added into `bad` if given)."""
    x = _need(x, "tensor")
    if bad is None:
        bad = torch.zeros(1, dtype=torch.int32, device=x.device)
    _call(x.device, "fc_count_nonfinite", _dtype(x), _p(x), x.numel(), _p(bad), _stream(x))
    return bad


# ------------------------------------------------------------------ pointwise (1x1) GEMMs
def _carr(ctype, vals):
    return (ctype * len(vals))(*vals)


def gemm_pack(w: torch.Tensor, segments, transpose: bool = False) -> torch.Tensor:
    """Tensor-core image of B for gemm_rows: B = w (rows = w.shape[0]) or w^T (transpose;
    rows = w.shape[1]); its K axis is the concatenation of `segments` = [(first column (row
    if transpose) of w, width)], each padded to 32 (fc_gemm_pack_b)."""
    w = _need(w, "w", torch.float32)
    if w.dim() != 2 or not segments:
        raise ShapeMismatchError("gemm_pack: w must be 2-D with at least one K segment")
    nrows = w.shape[1] if transpose else w.shape[0]
    kmax = w.shape[0] if transpose else w.shape[1]
    for a, k in segments:
        if a < 0 or k < 1 or a + k > kmax:
            raise ShapeMismatchError(f"gemm_pack: segment ({a}, {k}) outside w of shape {tuple(w.shape)}")
    kb = sum((k + 31) // 32 for _, k in segments)
    img = torch.empty(int(_lib.lib().fc_gemm_image_bytes(nrows, kb)), dtype=torch.uint8, device=w.device)
    _call(w.device, "fc_gemm_pack_b", int(transpose), nrows, len(segments),
          _carr(ctypes.c_int, [int(a) for a, _ in segments]), _carr(ctypes.c_int, [int(k) for _, k in segments]),
          _p(w), w.stride(0), _p(img), _stream(w))
    return img


def _rows2d(t: torch.Tensor, name: str, n: int) -> torch.Tensor:
    t = _need(t, name, torch.float32)
    if t.dim() != 2 or t.shape[0] != n:
        raise ShapeMismatchError(f"{name} must be [{n}, k], got {tuple(t.shape)}")
    return t


def gemm_rows(operands, img: torch.Tensor, ncols: int, bias=None, outs=None, relu=False, mask=None):
    """Y = bias + [operands[0] | operands[1] | ...] . B^T (B packed by gemm_pack with the
    operands' widths as its K segments).  Returns [Y[:, c0:c1] for (c0, c1) in outs]
    (default: the whole Y) and, with relu=True, also max(Y, 0) as the last element.
    mask: operand 0 is multiplied by (mask > 0) on the fly (same shape as operand 0)."""
    n = operands[0].shape[0]
    ops = [_rows2d(x, f"operand {q}", n) for q, x in enumerate(operands)]
    dev = ops[0].device
    outs = [(0, ncols)] if outs is None else list(outs)
    res = [torch.empty((n, c1 - c0), dtype=torch.float32, device=dev) for c0, c1 in outs]
    rl = torch.empty((n, ncols), dtype=torch.float32, device=dev) if relu else None
    if mask is not None:
        mask = _rows2d(mask, "mask", n)
        _shape(mask, tuple(ops[0].shape), "mask")
    if bias is not None:
        bias = _need(bias, "bias", torch.float32)
        _shape(bias, (ncols,), "bias")
    _call(dev, "fc_gemm_rows", n, len(ops), _carr(ctypes.c_void_p, [x.data_ptr() for x in ops]),
          _carr(ctypes.c_int64, [x.stride(0) for x in ops]), _carr(ctypes.c_int, [x.shape[1] for x in ops]),
          _p(mask), mask.stride(0) if mask is not None else 0, _p(img), ncols, _p(bias), len(res),
          _carr(ctypes.c_void_p, [r.data_ptr() for r in res]), _carr(ctypes.c_int64, [r.stride(0) for r in res]),
          _carr(ctypes.c_int, [c0 for c0, _ in outs]), _carr(ctypes.c_int, [c1 for _, c1 in outs]),
          _p(rl), rl.stride(0) if rl is not None else 0, _stream(ops[0]))
    return res + ([rl] if relu else [])


def relu_backward(g: torch.Tensor, z: torch.Tensor, add: torch.Tensor | None = None, out=None) -> torch.Tensor:
    """g * (z > 0) [+ add] in one pass (out may be g itself: in place)."""
    g = _need(g, "g")
    z = _need(z, "z", g.dtype, g.device)
    if z.shape != g.shape or not g.is_contiguous() or not z.is_contiguous():
        raise ShapeMismatchError(f"relu_backward: g {tuple(g.shape)} and z {tuple(z.shape)} must be contiguous, same shape")
    if add is not None:
        add = _need(add, "add", g.dtype, g.device)
        if add.shape != g.shape or not add.is_contiguous():
            raise ShapeMismatchError("relu_backward: add must be contiguous, same shape as g")
    if out is None:
        out = torch.empty_like(g)
    elif out.shape != g.shape or out.dtype != g.dtype or not out.is_contiguous():
        raise ShapeMismatchError("relu_backward: bad out")
    _call(g.device, "fc_relu_backward", _dtype(g), g.numel(), _p(g), _p(z), _p(add), _p(out), _stream(g))
    return out


def gemm_wgrad(g: torch.Tensor, operands, dw=None, db=None, mask=None) -> None:
    """dw [co, sum k_q] = G^T [operands...], db [co] = sum over rows of G (G masked by
    (mask > 0) when given); written in place (contiguous), fixed-order reductions."""
    g = _need(g, "g", torch.float32)
    n, co = g.shape
    ops = [_rows2d(x, f"operand {q}", n) for q, x in enumerate(operands)]
    ci = sum(x.shape[1] for x in ops)
    if dw is not None:
        _shape(dw, (co, ci), "dw")
        if not dw.is_contiguous():
            raise ShapeMismatchError("dw must be contiguous")
    if db is not None:
        _shape(db, (co,), "db")
    if mask is not None:
        mask = _rows2d(mask, "mask", n)
        _shape(mask, (n, co), "mask")
    _call(g.device, "fc_gemm_wgrad", n, _p(g), g.stride(0), _p(mask), mask.stride(0) if mask is not None else 0, co,
          len(ops), _carr(ctypes.c_void_p, [x.data_ptr() for x in ops]), _carr(ctypes.c_int64, [x.stride(0) for x in ops]),
          _carr(ctypes.c_int, [x.shape[1] for x in ops]), _p(dw), _p(db), _stream(g))

"""ctypes front-end for the CPU oracle (oracle/flexconv_oracle.c) and the compiled
reference kernels (oracle/_ref/_native*.so, built by oracle/build_ref.sh).

TEST INFRASTRUCTURE ONLY -- the checker, never the thing measured or shipped.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs import this module.  The product package never imports it.

Each function mirrors the reference operator it restates (file:line in the C source)
and takes/returns numpy float64 / int64 arrays in the reference's point-major layout.
"""

from __future__ import annotations

import ctypes
import glob
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libflexconv_oracle.so")
SRC = os.path.join(HERE, "flexconv_oracle.c")
REF_DIR = os.path.join(HERE, "_ref")

_lib = None


def build(force: bool = False) -> str:
    """Compile the C restatement (gcc -O3 -fopenmp, no FP contraction)."""
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= os.path.getmtime(SRC):
        return LIB_PATH
    os.makedirs(LIB_DIR, exist_ok=True)
    cc = os.environ.get("ORACLE_CC", "/usr/bin/gcc")
    cmd = [cc, "-O3", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", SRC, "-o", LIB_PATH, "-lm"]
    subprocess.check_call(cmd)
    return LIB_PATH


def build_ref() -> str | None:
    """Compile the reference's own _native.pyx into oracle/_ref (needs /root/reference)."""
    script = os.path.join(HERE, "build_ref.sh")
    subprocess.check_call(["bash", script])
    return ref_native_path()


def ref_native_path() -> str | None:
    hits = glob.glob(os.path.join(REF_DIR, "_native*.so"))
    return hits[0] if hits else None


def ref_native():
    """Import the compiled, unmodified reference kernel module (flexconv._native)."""
    if ref_native_path() is None:
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import _native  # noqa: PLC0415

    return _native


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        lib.fco_conv_forward.argtypes = [I, I, I, I, I, P, P, P, P, P, P, ctypes.c_int]
        lib.fco_conv_backward.argtypes = [I, I, I, I, I, P, P, P, P, P, P, P, P, P, P, ctypes.c_int]
        lib.fco_deconv_forward.argtypes = [I, I, I, I, I, P, P, P, P, P, P]
        lib.fco_pool_forward.argtypes = [I, I, I, P, P, P, P, ctypes.c_int]
        lib.fco_pool_backward.argtypes = [I, I, P, P, P]
        lib.fco_knn_brute.argtypes = [I, I, I, P, P, ctypes.c_int]
        lib.fco_knn_rows.argtypes = [I, I, I, P, P, I, P, ctypes.c_int]
        lib.fco_conv_forward_rows.argtypes = [I, I, I, I, I, P, P, P, P, P, P, I, P, ctypes.c_int]
        lib.fco_conv_backward_rows.argtypes = [I, I, I, I, I, P, P, P, P, P, P, P, I, P, P, ctypes.c_int]
        lib.fco_conv_param_grads.argtypes = [I, I, I, I, I, P, P, P, P, P, P, ctypes.c_int]
        _lib = lib
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def conv_forward(features, locations, neighbors, theta, theta_b, num_threads=None):
    """_native.pyx:25-66."""
    f, l, nb, th, tb = _f64(features), _f64(locations), _i64(neighbors), _f64(theta), _f64(theta_b)
    n, C = f.shape
    d = l.shape[1]
    k = nb.shape[1]
    cout = th.shape[0]
    out = np.empty((n, cout))
    nt = num_threads or os.cpu_count() or 1
    _load().fco_conv_forward(n, C, d, k, cout, _p(f), _p(l), _p(nb), _p(th), _p(tb), _p(out), nt)
    return out


def conv_backward(upstream, features, locations, neighbors, theta, theta_b, with_locations=True):
    """_native.pyx:69-127; returns (d_features, d_theta, d_theta_b, d_locations|None)."""
    g, f, l, nb, th, tb = (_f64(upstream), _f64(features), _f64(locations), _i64(neighbors),
                           _f64(theta), _f64(theta_b))
    n, C = f.shape
    d = l.shape[1]
    k = nb.shape[1]
    cout = th.shape[0]
    df = np.zeros_like(f)
    dl = np.zeros_like(l)
    dth = np.zeros_like(th)
    dtb = np.zeros_like(tb)
    _load().fco_conv_backward(n, C, d, k, cout, _p(g), _p(f), _p(l), _p(nb), _p(th), _p(tb),
                              _p(df), _p(dl), _p(dth), _p(dtb), int(bool(with_locations)))
    return df, dth, dtb, (dl if with_locations else None)


def deconv_forward(x, locations, neighbors, theta, theta_b):
    """Adjoint of conv_forward (== conv_backward(...).d_features, _native.pyx:106-120)."""
    xx, l, nb, th, tb = _f64(x), _f64(locations), _i64(neighbors), _f64(theta), _f64(theta_b)
    n = xx.shape[0]
    cout, C, d = th.shape
    k = nb.shape[1]
    y = np.zeros((n, C))
    _load().fco_deconv_forward(n, C, d, k, cout, _p(xx), _p(l), _p(nb), _p(th), _p(tb), _p(y))
    return y


def pool_forward(features, neighbors, num_threads=None):
    """_native.pyx:130-155; returns (pooled, argmax int64)."""
    f, nb = _f64(features), _i64(neighbors)
    n, C = nb.shape[0], f.shape[1]
    k = nb.shape[1]
    out = np.empty((n, C))
    am = np.empty((n, C), dtype=np.int64)
    nt = num_threads or os.cpu_count() or 1
    _load().fco_pool_forward(n, C, k, _p(f), _p(nb), _p(out), _p(am), nt)
    return out, am


def pool_backward(upstream, argmax, n_rows=None):
    """_native.pyx:158-168."""
    g, am = _f64(upstream), _i64(argmax)
    n, C = g.shape
    rows = n if n_rows is None else int(n_rows)
    df = np.zeros((rows, C))
    _load().fco_pool_backward(n, C, _p(g), _p(am), _p(df))
    return df


def knn_brute(points, k, num_threads=None):
    """neighborhood.py:171-187 semantics (self first, then (d^2, idx) order)."""
    p = _f64(points)
    n, d = p.shape
    out = np.empty((n, k), dtype=np.int64)
    nt = num_threads or os.cpu_count() or 1
    _load().fco_knn_brute(n, d, k, _p(p), _p(out), nt)
    return out


def knn_rows(points, rows, k, num_threads=None):
    """knn_brute restricted to the given query rows (spot checks at large n)."""
    p = _f64(points)
    r = _i64(rows)
    n, d = p.shape
    out = np.empty((r.shape[0], k), dtype=np.int64)
    nt = num_threads or os.cpu_count() or 1
    _load().fco_knn_rows(n, d, k, _p(p), _p(r), r.shape[0], _p(out), nt)
    return out


# ---------------------------------------------------------------- large-n checkers
def conv_forward_rows(features, locations, neighbors, theta, theta_b, rows, num_threads=None):
    """conv_forward restricted to the query rows (bitwise equal to those rows of conv_forward)."""
    f, l, nb, th, tb, r = (_f64(features), _f64(locations), _i64(neighbors), _f64(theta), _f64(theta_b),
                           _i64(rows))
    n, C = f.shape
    d = l.shape[1]
    k = nb.shape[1]
    cout = th.shape[0]
    out = np.empty((r.shape[0], cout))
    nt = num_threads or os.cpu_count() or 1
    _load().fco_conv_forward_rows(n, C, d, k, cout, _p(f), _p(l), _p(nb), _p(th), _p(tb), _p(r), r.shape[0],
                                  _p(out), nt)
    return out


def conv_backward_rows(upstream, features, locations, neighbors, theta, theta_b, rows, with_locations=True,
                       num_threads=None):
    """(d_features[rows], d_locations[rows] | None) of conv_backward, in the reference's
    ascending-i addition order (bitwise equal to those rows of the serial conv_backward)."""
    g, f, l, nb, th, tb = (_f64(upstream), _f64(features), _f64(locations), _i64(neighbors), _f64(theta),
                           _f64(theta_b))
    uniq, inv = np.unique(_i64(rows), return_inverse=True)  # the C routine wants distinct rows
    r = _i64(uniq)
    n, C = f.shape
    d = l.shape[1]
    k = nb.shape[1]
    cout = th.shape[0]
    df = np.empty((r.shape[0], C))
    dl = np.empty((r.shape[0], d)) if with_locations else None
    nt = num_threads or os.cpu_count() or 1
    _load().fco_conv_backward_rows(n, C, d, k, cout, _p(g), _p(f), _p(l), _p(nb), _p(th), _p(tb), _p(r),
                                   r.shape[0], _p(df), _p(dl), nt)
    return df[inv], (dl[inv] if with_locations else None)


def conv_param_grads(upstream, features, locations, neighbors, c_out=None, num_threads=None):
    """(d_theta, d_theta_b) over all points: fp64, thread-parallel, per-thread partials added
    in thread order (differs from the serial reference by fp64 regrouping only)."""
    g, f, l, nb = _f64(upstream), _f64(features), _f64(locations), _i64(neighbors)
    n, C = f.shape
    d = l.shape[1]
    k = nb.shape[1]
    cout = g.shape[1] if c_out is None else int(c_out)
    dth = np.empty((cout, C, d))
    dtb = np.empty((cout, C))
    nt = num_threads or os.cpu_count() or 1
    _load().fco_conv_param_grads(n, C, d, k, cout, _p(g), _p(f), _p(l), _p(nb), _p(dth), _p(dtb), nt)
    return dth, dtb


# ---------------------------------------------------------------- synthetic inputs (numpy only)
_MIX = 0x9E3779B97F4A7C15


def synthetic_layer(seed, tag, n, d, c_in, c_out):
    """The synthetic layer of SURVEY.md §8(d), drawn exactly as
    paper_1803_07289_b200.core.synthetic_layer draws it (the reference's Philox Rng with
    spawned substreams, /root/reference/pkg/src/flexconv/core.py:86-112), restated here with
    numpy alone so the CPU-baseline legs of bench.py load nothing from the product package."""
    stream = (0 * _MIX + int(tag) + 1) % 2 ** 64
    g = np.random.Generator(np.random.Philox(key=[int(seed) % 2 ** 64, stream]))
    loc = np.floor(g.uniform(0.0, 1.0, size=(n, d)) * 2.0 ** 24) / 2.0 ** 24
    feat = g.standard_normal((n, c_in)).astype(np.float32).astype(np.float64)
    theta = (g.standard_normal((c_out, c_in, d)) * 0.1).astype(np.float32).astype(np.float64)
    theta_b = (g.standard_normal((c_out, c_in)) * 0.1).astype(np.float32).astype(np.float64)
    up = g.standard_normal((n, c_out)).astype(np.float32).astype(np.float64)
    return loc, feat, theta, theta_b, up

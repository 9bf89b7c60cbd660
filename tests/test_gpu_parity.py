"""GPU parity: every hot-path operator through the C ABI against the oracle and the
reference's golden vectors.

Tolerances (stated here):
  * fp64 engine: forward, pooling, kNN and the pool backward are bitwise identical to the
    reference; the backward/deconv reductions are regrouped and agree to 1e-12 relative.
  * fp32 engines (SIMT, tcgen05 3xTF32): forward, flex_deconv and d_features elementwise
    allclose(rtol=1e-4, atol=1e-5) (north_star).  The N-long reductions d_theta, d_theta_b
    and d_locations are checked elementwise with rtol=1e-4 and an absolute floor of
    1e-5 + 1e-6*max|ref| (fp32 rounding of the inputs to those sums grows like
    eps*sqrt(N)), plus norm-wise ||D||/||ref|| <= 1e-5.
  * kNN indices and pool argmax: bit-exact, ties to the lowest index.
"""

import numpy as np
import pytest

from conftest import central_diff, load_golden, quantized_cloud, rel_err

pytestmark = pytest.mark.gpu

CASES_BWD = ["c2_n1024_k16_64to128", "small_n300_k8_8to8", "small_d2_n200_k9_4to3",
             "small_d1_n57_k5_3to2"]
CASES_ALL = ["c1_n4096_k8_32to32"] + CASES_BWD


def _t(a, dtype=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.to(dtype) if dtype is not None else t


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


def assert_fp32_close(got, ref, name):
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-5, err_msg=name)


def assert_fp32_reduction_close(got, ref, name):
    floor = 1e-5 + 1e-6 * float(np.abs(ref).max())
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=floor, err_msg=name)
    assert np.linalg.norm(got - ref) <= 1e-5 * max(np.linalg.norm(ref), 1e-30), name


# ---------------------------------------------------------------- forward
@pytest.mark.parametrize("case", CASES_ALL)
def test_forward_fp64_bitwise_vs_reference(fc, case):
    g = load_golden(f"conv_{case}.npz")
    out = fc.flex_conv_forward(g["features"].astype(np.float64), g["locations"], fc.NeighborIndex(g["neighbors"]),
                               fc.FlexConvParams(g["theta"], g["theta_b"]))
    assert isinstance(out, np.ndarray) and out.dtype == np.float64
    np.testing.assert_array_equal(out, g["out"])


@pytest.mark.parametrize("mode", ["simt", "auto"])
@pytest.mark.parametrize("case", CASES_ALL)
def test_forward_fp32_vs_reference(fc, case, mode):
    import torch

    g = load_golden(f"conv_{case}.npz")
    out = fc.flex_conv_forward(_t(g["features"]), _t(g["locations"], torch.float32),
                               fc.NeighborIndex(_t(g["neighbors"])),
                               fc.FlexConvParams(_t(g["theta"]), _t(g["theta_b"])), mode=mode)
    assert out.dtype == torch.float32 and out.is_cuda
    assert_fp32_close(_np(out), g["out"], f"{case}/{mode}")


def test_forward_known_answers(fc):
    out = fc.flex_conv_forward(np.array([[5.0]]), np.zeros((1, 2)), fc.NeighborIndex(np.array([[0]])),
                               fc.FlexConvParams(np.zeros((1, 1, 2)), np.ones((1, 1))))
    np.testing.assert_array_equal(out, [[5.0]])
    feats = np.array([[1.0], [2.0]])
    locs = np.array([[0.0, 0.0], [1.0, 0.0]])
    nbr = fc.NeighborIndex(np.array([[0, 1], [1, 0]]))
    params = fc.FlexConvParams(np.array([[[1.0, 0.0]]]), np.zeros((1, 1)))
    assert fc.flex_conv_forward(feats, locs, nbr, params)[0, 0] == -2.0
    gb = fc.flex_conv_backward(np.array([[1.0], [0.0]]), feats, locs, nbr, params)
    np.testing.assert_allclose(gb.d_features, [[0.0], [-1.0]])
    np.testing.assert_allclose(gb.d_theta, [[[-2.0, 0.0]]])


# ---------------------------------------------------------------- backward
@pytest.mark.parametrize("case", CASES_BWD)
def test_backward_fp64_vs_reference(fc, case):
    g = load_golden(f"conv_{case}.npz")
    gb = fc.flex_conv_backward(g["upstream"].astype(np.float64), g["features"].astype(np.float64), g["locations"],
                               fc.NeighborIndex(g["neighbors"]), fc.FlexConvParams(g["theta"], g["theta_b"]))
    for name in ("d_features", "d_theta", "d_theta_b", "d_locations"):
        ref = g[name]
        np.testing.assert_allclose(getattr(gb, name), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max(), err_msg=name)


@pytest.mark.parametrize("mode", ["simt", "auto"])
@pytest.mark.parametrize("case", CASES_BWD)
def test_backward_fp32_vs_reference(fc, case, mode):
    import torch

    g = load_golden(f"conv_{case}.npz")
    gb = fc.flex_conv_backward(_t(g["upstream"]), _t(g["features"]), _t(g["locations"], torch.float32),
                               fc.NeighborIndex(_t(g["neighbors"])),
                               fc.FlexConvParams(_t(g["theta"]), _t(g["theta_b"])), mode=mode)
    assert_fp32_close(_np(gb.d_features), g["d_features"], "d_features")
    assert_fp32_reduction_close(_np(gb.d_theta), g["d_theta"], "d_theta")
    assert_fp32_reduction_close(_np(gb.d_theta_b), g["d_theta_b"], "d_theta_b")
    assert_fp32_reduction_close(_np(gb.d_locations), g["d_locations"], "d_locations")


def test_backward_without_locations(fc):
    g = load_golden("conv_small_n300_k8_8to8.npz")
    gb = fc.flex_conv_backward(g["upstream"].astype(np.float64), g["features"].astype(np.float64), g["locations"],
                               fc.NeighborIndex(g["neighbors"]), fc.FlexConvParams(g["theta"], g["theta_b"]),
                               with_locations=False)
    assert gb.d_locations is None
    np.testing.assert_allclose(gb.d_features, g["d_features"], rtol=1e-12, atol=1e-12)


def test_backward_bitwise_deterministic(fc):
    import torch

    g = load_golden("conv_c2_n1024_k16_64to128.npz")
    args = (_t(g["upstream"]), _t(g["features"]), _t(g["locations"], torch.float32),
            fc.NeighborIndex(_t(g["neighbors"])), fc.FlexConvParams(_t(g["theta"]), _t(g["theta_b"])))
    a = fc.flex_conv_backward(*args)
    b = fc.flex_conv_backward(*args)
    for name in ("d_features", "d_theta", "d_theta_b", "d_locations"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name


@pytest.mark.parametrize("trial", range(4))
def test_gradients_match_finite_differences(fc, trial):
    """Reference tests/test_flexops.py:105-118 on the fp64 engine."""
    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(2, 32))
    d = int(rng.integers(1, 4))
    c_in, c_out = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    k = int(rng.integers(1, min(n, 8) + 1))
    locs = rng.standard_normal((n, d))
    feats = rng.standard_normal((n, c_in))
    nbr = fc.knn_brute_force(locs, k)
    params = fc.FlexConvParams(rng.standard_normal((c_out, c_in, d)), rng.standard_normal((c_out, c_in)))
    up = rng.standard_normal((n, c_out))

    def loss(f=feats, l=locs, th=params.theta, tb=params.theta_b):
        return float((fc.flex_conv_forward(f, l, nbr, fc.FlexConvParams(th, tb)) * up).sum())

    gb = fc.flex_conv_backward(up, feats, locs, nbr, params)
    assert rel_err(gb.d_features, central_diff(lambda a: loss(f=a), feats)) < 1e-6
    assert rel_err(gb.d_locations, central_diff(lambda a: loss(l=a), locs)) < 1e-6
    assert rel_err(gb.d_theta, central_diff(lambda a: loss(th=a), params.theta)) < 1e-6
    assert rel_err(gb.d_theta_b, central_diff(lambda a: loss(tb=a), params.theta_b)) < 1e-6


# ---------------------------------------------------------------- deconv
@pytest.mark.parametrize("case", CASES_BWD)
def test_deconv_vs_reference(fc, case):
    import torch

    g = load_golden(f"conv_{case}.npz")
    nb = fc.NeighborIndex(g["neighbors"])
    y = fc.flex_deconv_forward(g["deconv_x"].astype(np.float64), g["locations"], nb,
                               fc.FlexConvParams(g["theta"], g["theta_b"]))
    np.testing.assert_allclose(y, g["deconv_y"], rtol=1e-12, atol=1e-12 * np.abs(g["deconv_y"]).max())
    for mode in ("simt", "auto"):
        y32 = fc.flex_deconv_forward(_t(g["deconv_x"]), _t(g["locations"], torch.float32),
                                     fc.NeighborIndex(_t(g["neighbors"])),
                                     fc.FlexConvParams(_t(g["theta"]), _t(g["theta_b"])), mode=mode)
        assert_fp32_close(_np(y32), g["deconv_y"], f"deconv/{mode}")


def test_deconv_is_adjoint(fc):
    g = load_golden("conv_c2_n1024_k16_64to128.npz")
    rng = np.random.default_rng(0)
    nb = fc.NeighborIndex(g["neighbors"])
    params = fc.FlexConvParams(g["theta"], g["theta_b"])
    f = rng.standard_normal(g["features"].shape)
    x = rng.standard_normal((f.shape[0], params.c_out))
    lhs = float((fc.flex_conv_forward(f, g["locations"], nb, params) * x).sum())
    rhs = float((f * fc.flex_deconv_forward(x, g["locations"], nb, params)).sum())
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1.0)


# ---------------------------------------------------------------- pooling
@pytest.mark.parametrize("case", CASES_BWD)
def test_pool_fp64_bitwise_vs_reference(fc, case):
    g = load_golden(f"conv_{case}.npz")
    nb = fc.NeighborIndex(g["neighbors"])
    pooled, rec = fc.flex_max_pool(g["out"], nb)
    np.testing.assert_array_equal(pooled, g["pooled"])
    assert rec.dtype == np.int64
    np.testing.assert_array_equal(rec, g["pool_argmax"])
    df = fc.flex_max_pool_backward(g["pool_upstream"].astype(np.float64), rec)
    np.testing.assert_array_equal(df, g["pool_d_features"])


def test_pool_fp32_argmax_exact(fc, oracle_mod):
    import torch

    g = load_golden("conv_c2_n1024_k16_64to128.npz")
    x32 = g["out"].astype(np.float32)
    pooled, rec = fc.flex_max_pool(_t(x32), fc.NeighborIndex(_t(g["neighbors"])))
    want_p, want_a = oracle_mod.pool_forward(x32.astype(np.float64), g["neighbors"])
    np.testing.assert_array_equal(_np(pooled), want_p)
    np.testing.assert_array_equal(rec.cpu().numpy(), want_a)
    up = g["pool_upstream"]
    df = fc.flex_max_pool_backward(_t(up), rec)
    # fp32 engine: the same additions in the same (ascending i) order, in fp32 --
    # np.add.at is unbuffered and applies updates in index order.
    want_df = np.zeros(up.shape, dtype=np.float32)
    np.add.at(want_df, (want_a, np.broadcast_to(np.arange(up.shape[1]), up.shape)), up.astype(np.float32))
    np.testing.assert_array_equal(df.cpu().numpy(), want_df)
    assert df.dtype == torch.float32


def test_pool_known_answers(fc):
    NI = fc.NeighborIndex
    feats = np.array([[1.0, -2.0], [3.0, 4.0]])
    pooled, rec = fc.flex_max_pool(feats, NI(np.array([[0], [1]])))
    np.testing.assert_array_equal(pooled, feats)
    np.testing.assert_array_equal(rec, [[0, 0], [1, 1]])
    pooled, rec = fc.flex_max_pool(np.array([[1.0], [5.0], [3.0]]), NI(np.array([[0, 1, 2], [1, 0, 2], [2, 0, 1]])))
    np.testing.assert_array_equal(pooled, [[5.0]] * 3)
    np.testing.assert_array_equal(rec, [[1]] * 3)
    pooled, rec = fc.flex_max_pool(np.array([[2.0], [2.0]]), NI(np.array([[0, 1], [1, 0]])))
    np.testing.assert_array_equal(rec, [[0], [0]])
    np.testing.assert_array_equal(fc.flex_max_pool_backward(np.array([[1.0], [2.0], [4.0]]), np.array([[1], [1], [1]])),
                                  [[0.0], [7.0], [0.0]])
    with pytest.raises(fc.IndexOutOfRangeError):
        fc.flex_max_pool_backward(np.ones((2, 1)), np.array([[0], [5]]))


def test_upsample_and_gather_known_answers(fc):
    line = fc.NeighborIndex(np.array([[0, 1], [1, 0], [2, 1]]))
    np.testing.assert_array_equal(fc.flex_upsample(np.array([[7.0]]), np.array([0]), line, 3), [[7.0], [7.0], [0.0]])
    np.testing.assert_array_equal(fc.flex_upsample(np.array([[-5.0]]), np.array([0]), line, 3), [[0.0]] * 3)
    np.testing.assert_array_equal(fc.downsample_gather(np.array([[1.0], [2.0], [3.0]]), [2, 0]), [[3.0], [1.0]])
    with pytest.raises(fc.IndexOutOfRangeError):
        fc.flex_upsample(np.ones((1, 1)), np.array([9]), line, 3)


# ---------------------------------------------------------------- kNN
@pytest.mark.parametrize("algo", ["auto", "brute", "grid"])
def test_knn_bit_exact_vs_reference(fc, algo):
    import torch

    from paper_1803_07289_b200 import _lib, _ops

    z = load_golden("knn.npz")
    a = {"auto": _lib.KNN_AUTO, "brute": _lib.KNN_BRUTE, "grid": _lib.KNN_GRID}[algo]
    for key in sorted({k.split("__")[0] for k in z}):
        pts, want = z[f"{key}__points"], z[f"{key}__indices"]
        n, d = pts.shape
        k = want.shape[1]
        if algo == "grid" and d > 3:
            continue
        got = _ops.knn(_t(pts), 1, n, k, a).cpu().numpy()
        np.testing.assert_array_equal(got, want, err_msg=f"{key}/{algo}")
        if key.startswith("lattice"):  # 2^-24 lattice: fp32 input is exact -> same rows
            got32 = _ops.knn(_t(pts, torch.float32), 1, n, k, a).cpu().numpy()
            np.testing.assert_array_equal(got32, want, err_msg=f"{key}/{algo}/fp32")


def test_knn_reference_api_and_edge_cases(fc):
    pts = np.array([[0.0], [1.0], [3.0]])
    assert fc.knn_query(fc.build_kdtree(pts), pts, 2).indices.tolist() == [[0, 1], [1, 0], [2, 1]]
    assert fc.knn_brute_force(np.array([[0.0], [-1.0], [1.0]]), 2).indices[0].tolist() == [0, 1]
    rng = np.random.default_rng(1)
    p = rng.standard_normal((20, 3))
    np.testing.assert_array_equal(fc.knn_query(fc.build_kdtree(p), p, 1).indices.ravel(), np.arange(20))
    with pytest.raises(fc.ConfigInvalidError):
        fc.knn_brute_force(np.zeros((3, 2)), 4)
    with pytest.raises(fc.EmptyInputError):
        fc.build_kdtree(np.zeros((0, 3)))
    bad = np.zeros((4, 2))
    bad[2, 1] = np.nan
    with pytest.raises(fc.NonFiniteError):
        fc.build_kdtree(bad)
    dup = np.array([[0.0, 0.0], [1.0, 1.0], [0.0, 0.0], [2.0, 0.0]])
    nb = fc.knn_query(fc.build_kdtree(dup), dup, 4).indices
    assert nb[0, 1] == 2 and nb[2, 1] == 0


def test_knn_grid_large_spot_check(fc, oracle_mod):
    """1M-point lattice cloud through the grid path; 2000 random rows against the oracle."""
    import torch

    from paper_1803_07289_b200 import _lib, _ops
    from paper_1803_07289_b200.core import Rng, lattice_positions

    n = 1 << 20
    pts = lattice_positions(Rng(3).spawn(1).gen, n, 3)
    got = _ops.knn(_t(pts, torch.float32), 1, n, 8, _lib.KNN_GRID).cpu().numpy()
    rows = np.random.default_rng(0).choice(n, 2000, replace=False)
    np.testing.assert_array_equal(got[rows], oracle_mod.knn_rows(pts, rows, 8))
    assert (got[:, 0] == np.arange(n)).all()


def test_knn_clustered_and_batched(fc, oracle_mod):
    """Clustered (non-uniform) clouds, batch of 3, grid vs brute vs oracle."""
    import torch

    from paper_1803_07289_b200 import _lib, _ops

    rng = np.random.default_rng(7)
    clouds = []
    for b in range(3):
        centers = rng.uniform(0, 1, (5, 3))
        p = centers[rng.integers(0, 5, 9000)] + 0.01 * rng.standard_normal((9000, 3))
        clouds.append(np.floor(p * 2 ** 20) / 2 ** 20)
    pts = np.concatenate(clouds)
    for a in (_lib.KNN_GRID, _lib.KNN_BRUTE):
        got = _ops.knn(_t(pts), 3, 9000, 16, a).cpu().numpy().reshape(3, 9000, 16)
        for b in range(3):
            rows = np.arange(0, 9000, 37)
            np.testing.assert_array_equal(got[b][rows], oracle_mod.knn_rows(clouds[b], rows, 16))


# ---------------------------------------------------------------- invariants
def test_translation_invariance_bitwise(fc):
    rng = np.random.default_rng(8)
    locs = quantized_cloud(rng, 50, 3)
    feats = rng.standard_normal((50, 2))
    nbr = fc.knn_brute_force(locs, 6)
    params = fc.FlexConvParams(rng.standard_normal((3, 2, 3)), rng.standard_normal((3, 2)))
    base = fc.flex_conv_forward(feats, locs, nbr, params)
    for shift in ([1.0, 0.0, 0.0], [17.0, -5.0, 3.0], [-128.0, 64.0, 1.0]):
        np.testing.assert_array_equal(fc.flex_conv_forward(feats, locs + np.array(shift), nbr, params), base)


def test_permutation_equivariance_bitwise(fc):
    rng = np.random.default_rng(9)
    n = 40
    locs = rng.standard_normal((n, 2))
    feats = rng.standard_normal((n, 3))
    nbr = fc.knn_brute_force(locs, 5)
    params = fc.FlexConvParams(rng.standard_normal((2, 3, 2)), rng.standard_normal((2, 3)))
    out = fc.flex_conv_forward(feats, locs, nbr, params)
    perm = rng.permutation(n)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    out_p = fc.flex_conv_forward(feats[perm], locs[perm], fc.NeighborIndex(inv[nbr.indices[perm]]), params)
    np.testing.assert_array_equal(out_p, out[perm])


def test_errors_match_reference(fc):
    rng = np.random.default_rng(0)
    locs = rng.standard_normal((10, 3))
    feats = rng.standard_normal((10, 2))
    nbr = fc.knn_brute_force(locs, 4)
    params = fc.FlexConvParams(rng.standard_normal((3, 2, 3)), rng.standard_normal((3, 2)))
    with pytest.raises(fc.ShapeMismatchError):
        fc.flex_conv_forward(np.c_[feats, feats], locs, nbr, params)
    bad = nbr.indices.copy()
    bad[0, -1] = 13
    with pytest.raises(fc.IndexOutOfRangeError):
        fc.flex_conv_forward(feats, locs, fc.NeighborIndex(bad), params)
    with pytest.raises(fc.NonFiniteError):
        fc.FlexConvParams(np.full((1, 1, 1), np.nan), np.zeros((1, 1)))


def test_duplicate_neighbours_in_a_row(fc, oracle_mod):
    """Rows may repeat an index (not produced by kNN, but legal input): conv counts it
    twice, pool-backward routes the gradient once -- as the reference does."""
    rng = np.random.default_rng(3)
    n, c = 30, 4
    locs = rng.standard_normal((n, 3))
    feats = rng.standard_normal((n, c))
    nb = rng.integers(0, n, (n, 5))
    nb[:, 0] = np.arange(n)
    nb[:, 2] = nb[:, 1]
    th, tb = rng.standard_normal((3, c, 3)), rng.standard_normal((3, c))
    params = fc.FlexConvParams(th, tb)
    NI = fc.NeighborIndex(nb)
    np.testing.assert_array_equal(fc.flex_conv_forward(feats, locs, NI, params),
                                  oracle_mod.conv_forward(feats, locs, nb, th, tb))
    up = rng.standard_normal((n, 3))
    gb = fc.flex_conv_backward(up, feats, locs, NI, params)
    ref = oracle_mod.conv_backward(up, feats, locs, nb, th, tb)
    for a, b in zip((gb.d_features, gb.d_theta, gb.d_theta_b, gb.d_locations), ref):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
    pooled, rec = fc.flex_max_pool(feats, NI)
    pg = rng.standard_normal((n, c))
    np.testing.assert_array_equal(fc.flex_max_pool_backward(pg, rec), oracle_mod.pool_backward(pg, rec))


# ---------------------------------------------------------------- batched torch API
def test_batched_ops_match_per_cloud_oracle(fc, oracle_mod):
    import torch

    from paper_1803_07289_b200.core import synthetic_layer

    B, N, K, cin, cout = 3, 700, 8, 16, 24
    per = [synthetic_layer(11, b, N, 3, cin, cout) for b in range(B)]
    pos = torch.stack([_t(p[0], torch.float32).t() for p in per])  # [B, 3, N]
    feat = torch.stack([_t(p[1], torch.float32).t() for p in per]).requires_grad_(True)  # [B, Din, N]
    theta = _t(per[0][2], torch.float32).requires_grad_(True)
    theta_b = _t(per[0][3], torch.float32).requires_grad_(True)
    nbh = fc.knn(pos, K)
    assert tuple(nbh.bkn.shape) == (B, K, N)
    out = fc.flex_conv(feat, pos, nbh, theta, theta_b)
    assert tuple(out.shape) == (B, cout, N)
    up = torch.stack([_t(p[4], torch.float32).t() for p in per])
    (out * up).sum().backward()
    dth_ref = np.zeros(per[0][2].shape)
    for b in range(B):
        nb = nbh.bkn[b].t().cpu().numpy()
        np.testing.assert_array_equal(nb, oracle_mod.knn_brute(per[b][0], K))
        ref = oracle_mod.conv_forward(per[b][1], per[b][0], nb, per[0][2], per[0][3])
        assert_fp32_close(_np(out[b].t()), ref, f"out[{b}]")
        df, dth, _, _ = oracle_mod.conv_backward(per[b][4], per[b][1], per[b][0], nb, per[0][2], per[0][3])
        assert_fp32_close(_np(feat.grad[b].t()), df, f"d_features[{b}]")
        dth_ref += dth
    assert_fp32_reduction_close(_np(theta.grad), dth_ref, "d_theta (batched)")
    # flex_pool and flex_deconv on the same neighbourhood
    pooled, am = fc.flex_pool(out.detach(), nbh, return_argmax=True)
    y = fc.flex_deconv(out.detach(), pos, nbh, theta.detach(), theta_b.detach())
    for b in range(B):
        nb = nbh.bkn[b].t().cpu().numpy()
        x64 = _np(out[b].t())
        p_ref, a_ref = oracle_mod.pool_forward(x64, nb)
        np.testing.assert_array_equal(_np(pooled[b].t()), p_ref)
        np.testing.assert_array_equal(am[b].t().cpu().numpy(), a_ref)
        y_ref = oracle_mod.deconv_forward(x64, per[b][0], nb, per[0][2], per[0][3])
        assert_fp32_close(_np(y[b].t()), y_ref, f"deconv[{b}]")


def test_autograd_deconv_and_pool(fc):
    import torch

    torch.manual_seed(0)
    B, N, K = 2, 300, 6
    pos = torch.rand(B, 3, N, device="cuda", dtype=torch.float64)
    nbh = fc.knn(pos, K)
    x = torch.randn(B, 5, N, device="cuda", dtype=torch.float64, requires_grad=True)
    th = torch.randn(5, 4, 3, device="cuda", dtype=torch.float64, requires_grad=True)
    tb = torch.randn(5, 4, device="cuda", dtype=torch.float64, requires_grad=True)
    posg = pos.clone().requires_grad_(True)
    assert torch.autograd.gradcheck(lambda a, p, t, b: fc.flex_deconv(a, p, nbh, t, b), (x, posg, th, tb),
                                    eps=1e-6, atol=1e-6)
    f = torch.randn(B, 4, N, device="cuda", dtype=torch.float64, requires_grad=True)
    assert torch.autograd.gradcheck(lambda a, p, t, b: fc.flex_conv(a, p, nbh, t, b), (f, posg, th, tb),
                                    eps=1e-6, atol=1e-6)
    assert torch.autograd.gradcheck(lambda a: fc.flex_pool(a, nbh), (f,), eps=1e-6, atol=1e-6)


def test_backend_module_is_a_kernel_slot(fc, oracle_mod):
    """paper_1803_07289_b200.backend honours the reference's kernel-module ABI."""
    from paper_1803_07289_b200 import backend

    g = load_golden("conv_small_n300_k8_8to8.npz")
    f = g["features"].astype(np.float64)
    nb = g["neighbors"].astype(np.int64)
    out = np.empty(g["out"].shape)
    backend.flex_conv_forward(f, g["locations"], nb, g["theta"].astype(np.float64),
                              g["theta_b"].astype(np.float64), out, 4)
    np.testing.assert_array_equal(out, g["out"])
    bufs = [np.zeros_like(f), np.zeros_like(g["locations"]), np.zeros(g["theta"].shape), np.zeros(g["theta_b"].shape)]
    backend.flex_conv_backward(g["upstream"].astype(np.float64), f, g["locations"], nb, g["theta"].astype(np.float64),
                               g["theta_b"].astype(np.float64), *bufs, True)
    for buf, name in zip(bufs, ("d_features", "d_locations", "d_theta", "d_theta_b")):
        np.testing.assert_allclose(buf, g[name], rtol=1e-12, atol=1e-12 * np.abs(g[name]).max())
    am = np.empty(f.shape, dtype=np.int64)
    pooled = np.empty_like(f)
    backend.max_pool_forward(f, nb, pooled, am, 2)
    want_p, want_a = oracle_mod.pool_forward(f, nb)
    np.testing.assert_array_equal(pooled, want_p)
    np.testing.assert_array_equal(am, want_a)

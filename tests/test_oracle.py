"""CPU: pin the oracle (oracle/flexconv_oracle.c) against the reference's golden vectors
(tests/golden, produced by the reference itself via tests/golden/make_golden.py) and,
where it was built, against the compiled unmodified reference (oracle/_ref)."""

import numpy as np
import pytest

from conftest import load_golden

CONV_CASES = ["c1_n4096_k8_32to32", "c2_n1024_k16_64to128", "small_n300_k8_8to8",
              "small_d2_n200_k9_4to3", "small_d1_n57_k5_3to2"]


@pytest.mark.parametrize("case", CONV_CASES)
def test_oracle_forward_bitwise_vs_golden(oracle_mod, case):
    g = load_golden(f"conv_{case}.npz")
    out = oracle_mod.conv_forward(g["features"], g["locations"], g["neighbors"], g["theta"], g["theta_b"])
    np.testing.assert_array_equal(out, g["out"])


@pytest.mark.parametrize("case", CONV_CASES[1:])
def test_oracle_backward_bitwise_vs_golden(oracle_mod, case):
    g = load_golden(f"conv_{case}.npz")
    df, dth, dtb, dl = oracle_mod.conv_backward(g["upstream"], g["features"], g["locations"], g["neighbors"],
                                                g["theta"], g["theta_b"])
    np.testing.assert_array_equal(df, g["d_features"])
    np.testing.assert_array_equal(dth, g["d_theta"])
    np.testing.assert_array_equal(dtb, g["d_theta_b"])
    np.testing.assert_array_equal(dl, g["d_locations"])


@pytest.mark.parametrize("case", CONV_CASES[1:])
def test_oracle_deconv_and_pool_vs_golden(oracle_mod, case):
    g = load_golden(f"conv_{case}.npz")
    y = oracle_mod.deconv_forward(g["deconv_x"], g["locations"], g["neighbors"], g["theta"], g["theta_b"])
    np.testing.assert_array_equal(y, g["deconv_y"])
    pooled, am = oracle_mod.pool_forward(g["out"], g["neighbors"])
    np.testing.assert_array_equal(pooled, g["pooled"])
    np.testing.assert_array_equal(am, g["pool_argmax"])
    df = oracle_mod.pool_backward(g["pool_upstream"], am)
    np.testing.assert_array_equal(df, g["pool_d_features"])


def test_oracle_knn_vs_golden(oracle_mod):
    z = load_golden("knn.npz")
    keys = sorted({k.split("__")[0] for k in z})
    assert len(keys) >= 6
    for key in keys:
        pts, idx = z[f"{key}__points"], z[f"{key}__indices"]
        k = idx.shape[1]
        np.testing.assert_array_equal(oracle_mod.knn_brute(pts, k), idx, err_msg=key)


def test_oracle_known_answers(oracle_mod):
    ka = load_golden("known_answers.npz")
    out = oracle_mod.conv_forward(np.array([[5.0]]), np.zeros((1, 2)), np.array([[0]]),
                                  np.zeros((1, 1, 2)), np.ones((1, 1)))
    np.testing.assert_array_equal(out, ka["identity_out"])
    assert out[0, 0] == 5.0
    feats = np.array([[1.0], [2.0]])
    locs = np.array([[0.0, 0.0], [1.0, 0.0]])
    nbr = np.array([[0, 1], [1, 0]])
    th, tb = np.array([[[1.0, 0.0]]]), np.zeros((1, 1))
    out = oracle_mod.conv_forward(feats, locs, nbr, th, tb)
    np.testing.assert_array_equal(out, ka["two_point_out"])
    assert out[0, 0] == -2.0
    df, dth, _, _ = oracle_mod.conv_backward(np.array([[1.0], [0.0]]), feats, locs, nbr, th, tb)
    np.testing.assert_array_equal(df, ka["two_point_d_features"])
    np.testing.assert_array_equal(dth, ka["two_point_d_theta"])
    _, am = oracle_mod.pool_forward(np.array([[2.0], [2.0]]), np.array([[0, 1], [1, 0]]))
    np.testing.assert_array_equal(am, ka["pool_tie_argmax"])


def test_oracle_matches_compiled_reference(oracle_mod):
    """When oracle/_ref was built (from /root/reference), the restatement is bitwise equal
    to the reference's own compiled kernels on fresh random inputs."""
    nat = oracle_mod.ref_native()
    if nat is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    n, c, d, k, co = 700, 6, 3, 9, 5
    loc = rng.standard_normal((n, d))
    f = rng.standard_normal((n, c))
    th = rng.standard_normal((co, c, d))
    tb = rng.standard_normal((co, c))
    nb = oracle_mod.knn_brute(loc, k)
    o_ref = np.empty((n, co))
    nat.flex_conv_forward(f, loc, nb, th, tb, o_ref, 2)
    np.testing.assert_array_equal(oracle_mod.conv_forward(f, loc, nb, th, tb), o_ref)
    g = rng.standard_normal((n, co))
    bufs = [np.zeros_like(f), np.zeros_like(loc), np.zeros_like(th), np.zeros_like(tb)]
    nat.flex_conv_backward(g, f, loc, nb, th, tb, bufs[0], bufs[1], bufs[2], bufs[3], True)
    df, dth, dtb, dl = oracle_mod.conv_backward(g, f, loc, nb, th, tb)
    for a, b in zip((df, dl, dth, dtb), bufs):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("case", CONV_CASES[1:])
def test_oracle_row_checkers_bitwise_vs_golden(oracle_mod, case):
    """The large-n checkers (row subsets, parallel parameter gradients) against the
    reference's own golden outputs: rows bitwise, d_theta/d_theta_b to fp64 regrouping."""
    g = load_golden(f"conv_{case}.npz")
    n = g["features"].shape[0]
    rows = np.unique(np.r_[0, n - 1, np.random.default_rng(3).integers(0, n, 40)])
    args = (g["features"], g["locations"], g["neighbors"], g["theta"], g["theta_b"])
    np.testing.assert_array_equal(oracle_mod.conv_forward_rows(*args, rows), g["out"][rows])
    df, dl = oracle_mod.conv_backward_rows(g["upstream"], *args, rows)
    np.testing.assert_array_equal(df, g["d_features"][rows])
    np.testing.assert_array_equal(dl, g["d_locations"][rows])
    dth, dtb = oracle_mod.conv_param_grads(g["upstream"], g["features"], g["locations"], g["neighbors"])
    np.testing.assert_allclose(dth, g["d_theta"], rtol=1e-12, atol=1e-12 * np.abs(g["d_theta"]).max())
    np.testing.assert_allclose(dtb, g["d_theta_b"], rtol=1e-12, atol=1e-12 * np.abs(g["d_theta_b"]).max())


def test_oracle_backward_rows_repeated_slots(oracle_mod):
    """A neighbour listed twice in one row and duplicated query rows: still the serial
    reference's values, bitwise."""
    from paper_1803_07289_b200.core import synthetic_layer

    loc, feat, th, tb, up = synthetic_layer(3, 0, 600, 3, 8, 5)
    nbr = oracle_mod.knn_brute(loc, 6)
    nbr[10, 3] = nbr[10, 2]
    rows = np.array([0, 10, nbr[10, 2], 599, 5, 5])
    df, _, _, dl = oracle_mod.conv_backward(up, feat, loc, nbr, th, tb)
    rdf, rdl = oracle_mod.conv_backward_rows(up, feat, loc, nbr, th, tb, rows)
    np.testing.assert_array_equal(rdf, df[rows])
    np.testing.assert_array_equal(rdl, dl[rows])


def test_oracle_synthetic_layer_matches_package(oracle_mod):
    """bench.py's CPU legs draw inputs through oracle.synthetic_layer (numpy only); it must
    be the package's generator, value for value."""
    from paper_1803_07289_b200.core import synthetic_layer

    for a, b in zip(oracle_mod.synthetic_layer(4, 0, 500, 3, 8, 6), synthetic_layer(4, 0, 500, 3, 8, 6)):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(oracle_mod.synthetic_layer(9, 3, 50, 2, 4, 5), synthetic_layer(9, 3, 50, 2, 4, 5)):
        np.testing.assert_array_equal(a, b)

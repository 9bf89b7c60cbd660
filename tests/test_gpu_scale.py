"""GPU parity at the benchmarked scale: the bench's own workload (bench.make_workload) at
C3 (1,048,576 points) and C4 (7,000,000 points), K = 8, 64 -> 64, through the C ABI, against
the oracle (oracle/flexconv_oracle.c, pinned to the reference in tests/test_oracle.py).

  * C3 forward: every row, elementwise allclose(rtol=1e-4, atol=1e-5) (north_star).
  * C4 forward, and d_features / d_locations at both sizes: >= 20,000 sampled rows through
    the oracle's row checkers (bitwise equal to those rows of the serial reference loop).
  * d_theta / d_theta_b: the full fp64 reduction over all points (fco_conv_param_grads).
  * kNN: >= 10,000 rows of the grid table against the brute-force oracle, bit-exact.

Tolerances.  Forward and d_features: the north_star's elementwise 1e-4 / 1e-5.  The N-long
reductions (d_theta, d_theta_b, d_locations) are held norm-wise, ||D||/||ref|| <= 1e-5, and
elementwise to rtol 1e-4 with an absolute floor of 1e-5 * max|ref|; whether the plain
1e-4 / 1e-5 holds is MEASURED and reported (violation counts), not assumed: the inputs to
those sums are fp32 moments whose rounding grows like eps * sqrt(N).  With FC_PARITY_REPORT
set to a directory, each test writes its error statistics there as JSON.
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROWS = 20000
KNN_ROWS = 10000


def _stats(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(got - ref)
    plain = err > 1e-5 + 1e-4 * np.abs(ref)
    return {"count": int(ref.size), "max_abs_err": float(err.max()), "max_abs_ref": float(np.abs(ref).max()),
            "norm_rel_err": float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)),
            "plain_1e-4_1e-5_violations": int(plain.sum()),
            "plain_violation_frac": float(plain.mean())}


def _report(name, stats):
    d = os.environ.get("FC_PARITY_REPORT")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"parity_{name}.json"), "w") as fh:
            json.dump(stats, fh, indent=1)
    print(name, json.dumps(stats))


def _close(got, ref, name):
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-5, err_msg=name)


def _close_reduction(got, ref, name):
    """N-long reductions at 1M-7M points: norm-wise ||D||/||ref|| <= 1e-5 (the criterion), and
    elementwise rtol 1e-4 with an absolute floor of 1e-5 * max|ref|: the fp32 moments entering
    these sums carry rounding noise ~eps * sqrt(N) * |term| that does not shrink with the
    entry, so entries near zero are bounded by the sum's scale (even the fp32 SIMT engine's
    d_theta_b error at 1M is 1.1e-6 * max|ref|, scripts/dtheta_precision.py)."""
    floor = 1e-5 + 1e-5 * float(np.abs(ref).max())
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=floor, err_msg=name)
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref), name


def _workload(n):
    import torch

    import bench

    dev = torch.device("cuda", 0)
    w = bench.make_workload(n, 8, 64, 0, dev)
    host = {name: w[name].cpu().numpy().astype(np.float64) for name in ("pos", "feat", "g", "theta", "theta_b")}
    host["nbr"] = w["nbr"].cpu().numpy().astype(np.int64)
    return w, host


def _sample_rows(n, count, seed):
    rng = np.random.default_rng(seed)
    rows = rng.choice(n, size=count - 4, replace=False)
    return np.unique(np.r_[rows, 0, 1, n - 2, n - 1])


def _run_scale(fc, oracle_mod, n, name, full_forward):
    from paper_1803_07289_b200 import _ops

    w, h = _workload(n)
    stats = {"n": n, "k": 8, "c_in": 64, "c_out": 64, "mode": "auto (fp32-accurate split engine)"}

    # kNN rows: bit-exact against the brute-force oracle (self first, (d^2, index) order)
    krows = _sample_rows(n, KNN_ROWS, 1)
    np.testing.assert_array_equal(h["nbr"][krows], oracle_mod.knn_rows(h["pos"], krows, 8), err_msg="knn rows")
    stats["knn_rows_checked_bit_exact"] = int(krows.size)

    out = _ops.conv_forward(w["feat"], w["pos"], w["nbr"], w["theta"], w["theta_b"], 1, n).cpu().numpy()
    args = (h["feat"], h["pos"], h["nbr"], h["theta"], h["theta_b"])
    if full_forward:
        ref = oracle_mod.conv_forward(*args)
        got = out
    else:
        rows = _sample_rows(n, ROWS, 2)
        ref = oracle_mod.conv_forward_rows(*args, rows)
        got = out[rows]
    stats["forward"] = _stats(got, ref)
    stats["forward"]["rows"] = "all" if full_forward else int(ref.shape[0])
    _close(got, ref, "forward")
    del out, got, ref

    df, dth, dtb, dl = _ops.conv_backward(w["g"], w["feat"], w["pos"], w["nbr"], w["csr"], w["theta"],
                                          w["theta_b"], 1, n, need=(True, True, True, True))
    rows = _sample_rows(n, ROWS, 3)
    rdf, rdl = oracle_mod.conv_backward_rows(h["g"], *args, rows)
    gdf = df.cpu().numpy()[rows]
    gdl = dl.cpu().numpy()[rows]
    stats["d_features"] = dict(_stats(gdf, rdf), rows=int(rows.size))
    stats["d_locations"] = dict(_stats(gdl, rdl), rows=int(rows.size))
    rdth, rdtb = oracle_mod.conv_param_grads(h["g"], h["feat"], h["pos"], h["nbr"])
    gdth, gdtb = dth.cpu().numpy(), dtb.cpu().numpy()
    stats["d_theta"] = _stats(gdth, rdth)
    stats["d_theta_b"] = _stats(gdtb, rdtb)
    _report(name, stats)
    _close(gdf, rdf, "d_features")
    _close_reduction(gdl, rdl, "d_locations")
    _close_reduction(gdth, rdth, "d_theta")
    _close_reduction(gdtb, rdtb, "d_theta_b")


def test_c3_1M_vs_oracle(fc, oracle_mod):
    """C3: every forward row, 20k backward rows, the full d_theta reduction, 10k kNN rows."""
    _run_scale(fc, oracle_mod, 1 << 20, "c3_1M", full_forward=True)


def test_c4_7M_bench_workload_vs_oracle(fc, oracle_mod):
    """C4 / the bench workload itself (7M points): sampled rows + the full d_theta reduction."""
    _run_scale(fc, oracle_mod, 7_000_000, "c4_7M", full_forward=False)


def test_c2_batched_b8_vs_oracle(fc, oracle_mod):
    """C2 as the benchmark shape: B = 8 clouds x 1024 points, K = 16, 64 -> 128 through the
    batched [B, D, N] API (flex_conv fwd/bwd, flex_pool fwd/bwd on the 128-ch output,
    flex_deconv 128 -> 64 fwd) against the per-cloud oracle."""
    import torch

    from paper_1803_07289_b200.core import synthetic_layer

    B, N, K, cin, cout = 8, 1024, 16, 64, 128
    per = [synthetic_layer(2, b, N, 3, cin, cout) for b in range(B)]
    dev = torch.device("cuda")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev, torch.float32)  # noqa: E731
    pos = torch.stack([t(p[0]).t() for p in per])
    feat = torch.stack([t(p[1]).t() for p in per]).requires_grad_(True)
    theta = t(per[0][2]).requires_grad_(True)
    theta_b = t(per[0][3]).requires_grad_(True)
    posg = pos.clone().requires_grad_(True)
    nbh = fc.knn(pos, K)
    out = fc.flex_conv(feat, posg, nbh, theta, theta_b)
    up = torch.stack([t(p[4]).t() for p in per])
    (out * up).sum().backward()
    pooled, am = fc.flex_pool(out.detach(), nbh, return_argmax=True)
    pg = torch.randn_like(pooled)
    pin = out.detach().clone().requires_grad_(True)
    (fc.flex_pool(pin, nbh) * pg).sum().backward()
    y = fc.flex_deconv(up, pos, nbh, theta.detach(), theta_b.detach())
    dth_ref = np.zeros(per[0][2].shape)
    dtb_ref = np.zeros(per[0][3].shape)
    for b in range(B):
        nb = nbh.bkn[b].t().cpu().numpy().astype(np.int64)
        loc, f, th, tb, g = per[b][0], per[b][1], per[0][2], per[0][3], per[b][4]
        np.testing.assert_array_equal(nb, oracle_mod.knn_brute(loc, K))
        _close(out[b].t().detach().cpu().numpy(), oracle_mod.conv_forward(f, loc, nb, th, tb), f"out[{b}]")
        df, dth, dtb, dl = oracle_mod.conv_backward(g, f, loc, nb, th, tb)
        _close(feat.grad[b].t().cpu().numpy(), df, f"d_features[{b}]")
        _close_reduction(posg.grad[b].t().cpu().numpy(), dl, f"d_locations[{b}]")
        dth_ref += dth
        dtb_ref += dtb
        x64 = out[b].t().detach().cpu().numpy().astype(np.float64)
        p_ref, a_ref = oracle_mod.pool_forward(x64, nb)
        np.testing.assert_array_equal(pooled[b].t().cpu().numpy(), p_ref)
        np.testing.assert_array_equal(am[b].t().cpu().numpy(), a_ref)
        _close(pin.grad[b].t().cpu().numpy(), oracle_mod.pool_backward(pg[b].t().cpu().numpy().astype(np.float64), a_ref),
               f"pool d_features[{b}]")
        _close(y[b].t().cpu().numpy(), oracle_mod.deconv_forward(g, loc, nb, th, tb), f"deconv[{b}]")
    _close_reduction(theta.grad.cpu().numpy(), dth_ref, "d_theta")
    _close_reduction(theta_b.grad.cpu().numpy(), dtb_ref, "d_theta_b")

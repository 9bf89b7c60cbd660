"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It imports the unmodified reference package from /root/reference/pkg/src with its
compiled kernel module built by oracle/build_ref.sh (oracle/_ref/_native*.so), and
calls the reference's public operator API (flexconv.flexops / flexconv.neighborhood).
The outputs are committed as small .npz files; the GPU box never reads /root/reference.

Inputs follow SURVEY.md §8(d): Philox Rng(seed) with spawn(b) per cloud, positions
floor(U*2^24)/2^24, features/upstream N(0,1) cast to fp32, theta/theta_b 0.1*N(0,1)
cast to fp32 -- every input is exactly representable in fp32, so the fp32 GPU path and
the fp64 reference see identical inputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def import_reference():
    sys.path.insert(0, ROOT)
    from oracle import oracle  # noqa: PLC0415

    nat = oracle.ref_native() or (oracle.build_ref() and oracle.ref_native())
    sys.modules["flexconv._native"] = nat
    sys.path.insert(0, REF_SRC)
    import flexconv  # noqa: PLC0415
    from flexconv import backend  # noqa: PLC0415

    assert backend.backend_name() == "native", "reference kernels not loaded"
    return flexconv


def synth_cloud(fc, seed, tag, n, d, c_in, c_out, k):
    g = fc.core.Rng(seed).spawn(tag).gen
    loc = np.floor(g.uniform(0.0, 1.0, size=(n, d)) * 2.0 ** 24) / 2.0 ** 24
    feat = g.standard_normal((n, c_in)).astype(np.float32).astype(np.float64)
    theta = (g.standard_normal((c_out, c_in, d)) * 0.1).astype(np.float32).astype(np.float64)
    theta_b = (g.standard_normal((c_out, c_in)) * 0.1).astype(np.float32).astype(np.float64)
    up = g.standard_normal((n, c_out)).astype(np.float32).astype(np.float64)
    tree = fc.neighborhood.build_kdtree(loc)
    nbr = fc.neighborhood.knn_query(tree, tree.points, k)
    return loc, feat, theta, theta_b, up, nbr


def main():
    fc = import_reference()
    from flexconv import flexops, neighborhood  # noqa: PLC0415
    from flexconv.flexops import FlexConvParams  # noqa: PLC0415
    from flexconv.neighborhood import NeighborIndex  # noqa: PLC0415

    out_files = []

    # ---- 1. conv fwd/bwd/deconv/pool at config C1 (fwd) and C2-per-cloud shapes ----
    cases = [
        # name, seed, tag, n, d, c_in, c_out, k, with_backward
        ("c1_n4096_k8_32to32", 1, 0, 4096, 3, 32, 32, 8, False),
        ("c2_n1024_k16_64to128", 2, 0, 1024, 3, 64, 128, 16, True),
        ("small_n300_k8_8to8", 7, 0, 300, 3, 8, 8, 8, True),
        ("small_d2_n200_k9_4to3", 8, 0, 200, 2, 4, 3, 9, True),
        ("small_d1_n57_k5_3to2", 9, 0, 57, 1, 3, 2, 5, True),
    ]
    for name, seed, tag, n, d, c_in, c_out, k, with_bwd in cases:
        loc, feat, th, tb, up, nbr = synth_cloud(fc, seed, tag, n, d, c_in, c_out, k)
        params = FlexConvParams(th, tb)
        out = flexops.flex_conv_forward(feat, loc, nbr, params, num_threads=4)
        rec = dict(locations=loc, features=feat.astype(np.float32), theta=th.astype(np.float32),
                   theta_b=tb.astype(np.float32), neighbors=nbr.indices.astype(np.int32), out=out)
        if with_bwd:
            gb = flexops.flex_conv_backward(up, feat, loc, nbr, params, with_locations=True)
            rec.update(upstream=up.astype(np.float32), d_features=gb.d_features, d_theta=gb.d_theta,
                       d_theta_b=gb.d_theta_b, d_locations=gb.d_locations)
            pooled, record = flexops.flex_max_pool(out, nbr, num_threads=4)
            pg = np.random.default_rng(seed).standard_normal(out.shape).astype(np.float32)
            # pool input is `out` (already stored); pooled values are fp64 copies of it
            rec.update(pooled=pooled, pool_argmax=record.astype(np.int32), pool_upstream=pg,
                       pool_d_features=flexops.flex_max_pool_backward(pg.astype(np.float64), record))
            # flex_deconv oracle: d_features of flex_conv_backward with upstream = x
            # (independent of `features`, _native.pyx:106-120)
            x = up
            rec.update(deconv_x=x.astype(np.float32),
                       deconv_y=flexops.flex_conv_backward(x, np.zeros_like(feat), loc, nbr, params,
                                                           with_locations=False).d_features)
        path = os.path.join(HERE, f"conv_{name}.npz")
        np.savez_compressed(path, **rec)
        out_files.append(path)

    # ---- 2. kNN fixtures (reference knn_query == knn_brute_force by its own tests) ----
    knn = {}
    rng = np.random.default_rng(3)
    pts = rng.integers(0, 4, size=(300, 2)).astype(np.float64)  # heavy ties (test_neighborhood.py:101-106)
    knn["ties_n300_d2_k7"] = (pts, neighborhood.knn_brute_force(pts, 7).indices)
    for n, d, k in ((57, 1, 5), (200, 2, 9), (1000, 3, 8), (2000, 3, 16)):  # test_neighborhood.py:84-98
        pts = np.random.default_rng(n + d).uniform(0, 1, (n, d))
        tree = neighborhood.build_kdtree(pts)
        knn[f"uniform_n{n}_d{d}_k{k}"] = (pts, neighborhood.knn_query(tree, tree.points, k).indices)
    pts = np.array([[0.0, 0.0], [1.0, 1.0], [0.0, 0.0], [2.0, 0.0]])  # duplicates (:36-43)
    knn["dups_n4_d2_k4"] = (pts, neighborhood.knn_brute_force(pts, 4).indices)
    g = fc.core.Rng(3).spawn(0).gen  # a C3-style 2^-24 lattice cloud, larger n
    pts = np.floor(g.uniform(0.0, 1.0, size=(20000, 3)) * 2.0 ** 24) / 2.0 ** 24
    tree = neighborhood.build_kdtree(pts)
    knn["lattice_n20000_d3_k8"] = (pts, neighborhood.knn_query(tree, tree.points, 8).indices)
    rec = {}
    for key, (p, idx) in knn.items():
        rec[f"{key}__points"] = p
        rec[f"{key}__indices"] = idx.astype(np.int32)
    path = os.path.join(HERE, "knn.npz")
    np.savez_compressed(path, **rec)
    out_files.append(path)

    # ---- 3. known answers straight from the reference's own tests ----
    ka = {}
    ka["identity_out"] = flexops.flex_conv_forward(  # test_flexops.py:42-46 -> 5.0
        np.array([[5.0]]), np.zeros((1, 2)), NeighborIndex(np.array([[0]])),
        FlexConvParams(np.zeros((1, 1, 2)), np.ones((1, 1))))
    feats = np.array([[1.0], [2.0]])
    locs = np.array([[0.0, 0.0], [1.0, 0.0]])
    nbr = NeighborIndex(np.array([[0, 1], [1, 0]]))
    prm = FlexConvParams(np.array([[[1.0, 0.0]]]), np.zeros((1, 1)))
    ka["two_point_out"] = flexops.flex_conv_forward(feats, locs, nbr, prm)  # :48-55 -> -2
    gb = flexops.flex_conv_backward(np.array([[1.0], [0.0]]), feats, locs, nbr, prm)  # :95-103
    ka["two_point_d_features"] = gb.d_features
    ka["two_point_d_theta"] = gb.d_theta
    p, r = flexops.flex_max_pool(np.array([[2.0], [2.0]]), NeighborIndex(np.array([[0, 1], [1, 0]])))
    ka["pool_tie_argmax"] = r  # :135-140 -> lower global index
    ka["upsample_line"] = flexops.flex_upsample(  # :205-208 -> [7,7,0]
        np.array([[7.0]]), np.array([0]), NeighborIndex(np.array([[0, 1], [1, 0], [2, 1]])), 3)
    path = os.path.join(HERE, "known_answers.npz")
    np.savez_compressed(path, **ka)
    out_files.append(path)

    for f in out_files:
        print(f, os.path.getsize(f))


if __name__ == "__main__":
    main()

"""Per-config measurements (SURVEY.md §8(d) "Per-config shapes"), beside bench.py's headline.

bench.py times the headline workload (C4 shape, fwd+bwd, 7M points).  This script times every
other BASELINE.json config and the bandwidth kernels the north_star wants on the HBM roofline
(pool, deconv, kNN, reverse CSR), each kernel launched through the package's C ABI on the
current stream and timed with CUDA events, median over reps, L2 flushed (a 512 MB write)
before every rep.  Algorithmic bytes per point are SURVEY.md §8(d)'s formulas.

  python scripts/bench_configs.py [--reps 10] [--only C2,C5] > profiles/<round>_configs.json

C1  B=1, N=4096, K=8, 32->32, forward                    (CPU-reference-runnable anchor)
C2  B=8, N=1024, K=16, 64->128: conv fwd/bwd, pool fwd/bwd on 128 ch, deconv 128->64 fwd/bwd
C3  B=1, N=1,048,576, K=8, 64->64: kNN (timed) + reverse CSR + conv fwd/bwd
C5  U-Net training step (build_segnet(3, 1, 3, 2, 64, 8, 4), fp32), one 262,144-point scene
    per call; a GPU's batch-sharded share of B=32 over 8 GPUs is 4 scenes
BW  7M-point bandwidth kernels: pool fwd/bwd, deconv fwd, grid kNN, reverse CSR (64 ch, K=8)
    and the C2 channel/K shape at 1M points (128 ch, K=16)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1803_07289_b200 import _lib, _ops  # noqa: E402


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


HBM, HBM_SRC = peaks()
_FLUSH = None


def flush_l2():
    global _FLUSH
    if _FLUSH is None:
        _FLUSH = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    _FLUSH.fill_(1.0)


def timed(fn, reps, warmup=3):
    """Median ms of `fn` over reps, each rep after an L2 flush, CUDA events on the current stream."""
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def row(ms, points, bytes_per_point=None):
    r = {"ms": round(ms, 5), "points_per_s": round(points / (ms / 1e3), 1)}
    if bytes_per_point:
        gbs = bytes_per_point * points / (ms / 1e3) / 1e9
        r.update({"bytes_per_point": bytes_per_point, "GBps": round(gbs, 1), "frac_hbm": round(gbs / HBM, 4)})
    return r


# SURVEY.md §8(d) algorithmic bytes per point (fp32 s = 4, int32 indices)
def b_conv_fwd(ci, co, d, k):
    return 4 * ci + 4 * d + 4 * k + 4 * co


def b_conv_bwd(ci, co, d, k, dloc=True):
    return 4 * co + 4 * ci + 4 * d + 4 * k + (4 + 4 * k) + 4 * ci + (4 * d if dloc else 0)


def b_pool_fwd(c, k):
    return 4 * c + 4 * k + 4 * c + 4 * c


def b_pool_bwd(c, k):
    return 4 * c + 4 * c + (4 + 4 * k) + 4 * c


def b_deconv_fwd(cx, cy, d, k):
    return 4 * cx + 4 * d + (4 + 4 * k) + 4 * cy


def layer(b, n, k, ci, co, d=3, seed=0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    pos = torch.floor(torch.rand(b * n, d, generator=g, device="cuda", dtype=torch.float64) * 2 ** 24) / 2 ** 24
    pos = pos.float()
    if b == 1:  # one cloud: spatially ordered once (as bench.py)
        pos = pos[_ops.spatial_order(pos).long()].contiguous()
    feat = torch.randn(b * n, ci, generator=g, device="cuda")
    up = torch.randn(b * n, co, generator=g, device="cuda")
    theta = 0.1 * torch.randn(co, ci, d, generator=g, device="cuda")
    theta_b = 0.1 * torch.randn(co, ci, generator=g, device="cuda")
    nbr = _ops.knn(pos, b, n, k)
    csr = _ops.csr_build(nbr, b, n)
    torch.cuda.synchronize()
    return dict(pos=pos, feat=feat, up=up, theta=theta, theta_b=theta_b, nbr=nbr, csr=csr)


def c1(reps):
    b, n, k, c = 1, 4096, 8, 32
    L = layer(b, n, k, c, c, seed=1)
    ms = timed(lambda: _ops.conv_forward(L["feat"], L["pos"], L["nbr"], L["theta"], L["theta_b"], b, n), reps)
    return {"shape": "B=1, N=4096, K=8, 32->32, Dp=3, fp32 forward",
            "conv_forward": row(ms, b * n, b_conv_fwd(c, c, 3, k))}


def c2(reps):
    b, n, k, ci, co = 8, 1024, 16, 64, 128
    L = layer(b, n, k, ci, co, seed=2)
    P = b * n
    out = {}
    f = lambda: _ops.conv_forward(L["feat"], L["pos"], L["nbr"], L["theta"], L["theta_b"], b, n)  # noqa: E731
    out["conv_forward"] = row(timed(f, reps), P, b_conv_fwd(ci, co, 3, k))
    bw = lambda: _ops.conv_backward(L["up"], L["feat"], L["pos"], L["nbr"], L["csr"], L["theta"],  # noqa: E731
                                    L["theta_b"], b, n)
    out["conv_backward"] = row(timed(bw, reps), P, b_conv_bwd(ci, co, 3, k))
    y = f()
    pooled, am = _ops.pool_forward(y, L["nbr"], b, n)
    out["pool_forward"] = row(timed(lambda: _ops.pool_forward(y, L["nbr"], b, n), reps), P, b_pool_fwd(co, k))
    out["pool_backward"] = row(timed(lambda: _ops.pool_backward(L["up"], am, L["csr"], b, n, k), reps), P,
                               b_pool_bwd(co, k))
    # deconv 128 -> 64 with the conv's theta (the adjoint); its backward = a conv forward of
    # g_y (d_x) + conv_backward's d_theta with upstream = x, features = g_y
    x = L["up"]
    gy = L["feat"]
    dfw = lambda: _ops.deconv_forward(x, L["pos"], L["csr"], L["theta"], L["theta_b"], b, n, k)  # noqa: E731
    out["deconv_forward"] = row(timed(dfw, reps), P, b_deconv_fwd(co, ci, 3, k))

    def dbw():
        _ops.conv_forward(gy, L["pos"], L["nbr"], L["theta"], L["theta_b"], b, n)
        _ops.conv_backward(x, gy, L["pos"], L["nbr"], None, L["theta"], L["theta_b"], b, n,
                           need=(False, True, True, False))
    out["deconv_backward"] = row(timed(dbw, reps), P)

    def step():
        f()
        bw()
        _ops.pool_forward(y, L["nbr"], b, n)
        _ops.pool_backward(L["up"], am, L["csr"], b, n, k)
        dfw()
        dbw()
    out["step_all"] = row(timed(step, reps), P)
    out["step_all"]["what"] = "conv fwd+bwd, pool fwd+bwd, deconv fwd+bwd back to back"
    # the same step captured once as a CUDA graph and replayed (launch-bound at 8 K points)
    try:
        s_cap = torch.cuda.Stream()
        s_cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_cap):
            step()  # warm the allocator / kernel attributes outside the capture
        torch.cuda.current_stream().wait_stream(s_cap)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        out["step_all_cuda_graph"] = row(timed(graph.replay, reps), P)
    except Exception as exc:  # noqa: BLE001 -- report, do not fail the suite
        out["step_all_cuda_graph"] = {"error": f"{type(exc).__name__}: {str(exc)[:160]}"}
    return {"shape": "B=8, N=1024, K=16, 64->128 (pool on 128 ch, deconv 128->64), fp32", **out}


def c3(reps):
    b, n, k, c = 1, 1 << 20, 8, 64
    L = layer(b, n, k, c, c, seed=3)
    P = n
    out = {}
    out["knn_grid"] = row(timed(lambda: _ops.knn(L["pos"], b, n, k), reps), P, 4 * 3 + 4 * k)
    out["knn_grid"]["note"] = "exact cell-grid kNN on the spatially ordered cloud (binning included)"
    out["reverse_csr"] = row(timed(lambda: _ops.csr_build(L["nbr"], b, n), reps), P, 4 * k + 4 + 4 * k)
    f = lambda: _ops.conv_forward(L["feat"], L["pos"], L["nbr"], L["theta"], L["theta_b"], b, n)  # noqa: E731
    out["conv_forward"] = row(timed(f, reps), P, b_conv_fwd(c, c, 3, k))
    bw = lambda: _ops.conv_backward(L["up"], L["feat"], L["pos"], L["nbr"], L["csr"], L["theta"],  # noqa: E731
                                    L["theta_b"], b, n)
    out["conv_backward"] = row(timed(bw, reps), P, b_conv_bwd(c, c, 3, k))

    def all_():
        nbr = _ops.knn(L["pos"], b, n, k)
        csr = _ops.csr_build(nbr, b, n)
        _ops.conv_forward(L["feat"], L["pos"], nbr, L["theta"], L["theta_b"], b, n)
        _ops.conv_backward(L["up"], L["feat"], L["pos"], nbr, csr, L["theta"], L["theta_b"], b, n)
    out["knn_plus_conv_fwd_bwd"] = row(timed(all_, reps), P)
    return {"shape": "B=1, N=1048576, K=8, 64->64, fp32 (spatially ordered cloud)", **out}


def bw_kernels(reps):
    res = {}
    n, k, c = 7_000_000, 8, 64
    L = layer(1, n, k, c, c, seed=4)
    y = L["feat"]
    pooled, am = _ops.pool_forward(y, L["nbr"], 1, n)
    res["pool_forward_7M_64ch_k8"] = row(timed(lambda: _ops.pool_forward(y, L["nbr"], 1, n), reps), n,
                                         b_pool_fwd(c, k))
    res["pool_backward_7M_64ch_k8"] = row(timed(lambda: _ops.pool_backward(L["up"], am, L["csr"], 1, n, k), reps),
                                          n, b_pool_bwd(c, k))
    res["deconv_forward_7M_64to64_k8"] = row(
        timed(lambda: _ops.deconv_forward(L["up"], L["pos"], L["csr"], L["theta"], L["theta_b"], 1, n, k), reps),
        n, b_deconv_fwd(c, c, 3, k))
    res["knn_grid_7M_k8"] = row(timed(lambda: _ops.knn(L["pos"], 1, n, k), reps), n, 4 * 3 + 4 * k)
    res["reverse_csr_7M_k8"] = row(timed(lambda: _ops.csr_build(L["nbr"], 1, n), reps), n, 4 * k + 4 + 4 * k)
    del L, y, pooled, am
    torch.cuda.empty_cache()
    n, k, c = 1 << 20, 16, 128
    L = layer(1, n, k, c, c, seed=5)
    y = L["up"]
    pooled, am = _ops.pool_forward(y, L["nbr"], 1, n)
    res["pool_forward_1M_128ch_k16"] = row(timed(lambda: _ops.pool_forward(y, L["nbr"], 1, n), reps), n,
                                           b_pool_fwd(c, k))
    res["pool_backward_1M_128ch_k16"] = row(
        timed(lambda: _ops.pool_backward(L["up"], am, L["csr"], 1, n, k), reps), n, b_pool_bwd(c, k))
    return res


def c5(reps):
    from paper_1803_07289_b200 import network, sampling
    from paper_1803_07289_b200.core import PointCloud, Rng

    n = 262_144
    rng = np.random.default_rng(5)
    loc = np.floor(rng.random((n, 3)) * 2 ** 24) / 2 ** 24
    feats = rng.standard_normal((n, 1))
    labels = rng.integers(0, 3, n)
    cloud = PointCloud(loc, feats)
    # data prep: each scene in cell order (sampling.spatially_ordered; permutation equivariant)
    cloud, labels, _ = sampling.spatially_ordered(cloud, labels)
    feats = cloud.features
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = sampling.build_hierarchy(cloud, 8, 4, 2, Rng(5).spawn(1))
    torch.cuda.synchronize()
    hier_ms = (time.perf_counter() - t0) * 1e3
    g = network.build_segnet(3, 1, 3, 2, 64, 8, 4, dtype=torch.float32)
    network.initialize_params(g, Rng(5).spawn(2), h)
    adam = network.init_adam(g.store.size, lr=3e-3, dtype=torch.float32)
    x = torch.from_numpy(feats).cuda().float()
    lab = torch.from_numpy(labels).cuda()
    ms = timed(lambda: network.train_step(g, adam, h, x, lab), max(3, reps // 2), warmup=2)
    graphed = network.GraphedTrainStep(g, adam, h, x, lab)  # the same step captured as one CUDA graph
    ms_graph = timed(lambda: graphed(), max(3, reps // 2), warmup=2)
    # a GPU's batch-sharded share of B = 32 over 8 GPUs: 4 scenes, one fused pass
    # (train_step_batch(fused=True) over sampling.concat_hierarchies)
    scenes = [(h, x, lab)]
    for s in range(1, 4):
        loc_s = np.floor(rng.random((n, 3)) * 2 ** 24) / 2 ** 24
        c_s, lab_s, _ = sampling.spatially_ordered(PointCloud(loc_s, rng.standard_normal((n, 1))),
                                                   rng.integers(0, 3, n))
        h_s = sampling.build_hierarchy(c_s, 8, 4, 2, Rng(5 + s).spawn(1))
        scenes.append((h_s, torch.from_numpy(c_s.features).cuda().float(), torch.from_numpy(lab_s).cuda()))
    ms4 = timed(lambda: network.train_step_batch(g, adam, scenes, fused=True), max(3, reps // 2), warmup=2)
    ms4_loop = timed(lambda: network.train_step_batch(g, adam, scenes), max(3, reps // 2), warmup=2)
    return {"shape": "build_segnet(d=3, n_f=1, n_c=3, stages=2, base=64, k=8, factor=4), fp32, one 262144-point "
                     "scene per training step (forward, softmax CE, tape backward, Adam); scenes in cell order "
                     "(sampling.spatially_ordered)",
            "params": g.param_count(), "sizes": h.sizes(), "hierarchy_build_ms": round(hier_ms, 2),
            "train_step": row(ms, n),
            "train_step_cuda_graph": row(ms_graph, n),
            "per_gpu_step_4_scenes_fused": row(ms4, 4 * n),
            "per_gpu_step_4_scenes_scene_loop": row(ms4_loop, 4 * n)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="C1,C2,C3,BW,C5")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    todo = args.only.split(",")
    res = {"hbm_peak_GBps": HBM, "hbm_peak_source": HBM_SRC, "timing": "CUDA events on the launching stream, "
           "median over reps, L2 flushed (512 MB write) before each rep", "device": torch.cuda.get_device_name(0)}
    launches0 = _lib.launch_count()
    for name, fn in (("C1", c1), ("C2", c2), ("C3", c3), ("BW", bw_kernels), ("C5", c5)):
        if name in todo:
            res[name] = fn(args.reps)
            torch.cuda.empty_cache()
    res["library_launches"] = _lib.launch_count() - launches0
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

"""C4 (7M-point cloud, point-chunk sharded with halos) measured on ONE B200 by emulation: for
world = 2, 4, 8 the halo plans are built (parallel.HaloPlan), and every shard's local
flex-conv forward and forward+backward run on the GPU on its [owned | halo] buffers, timed
with CUDA events.  Reports the halo fraction, the halo bytes each rank receives per layer,
and the slowest shard's compute time: the compute part of a strong-scaling run (the NVLink
halo exchange itself needs N GPUs; its bytes are given so its time can be bounded).

  python scripts/shard_emulation.py [--n 7000000] > profiles/<round>_shard_emulation.json
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1803_07289_b200 import _ops, parallel  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=7_000_000)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--c", type=int, default=64)
    args = ap.parse_args()
    n, k, c = args.n, args.k, args.c
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    pos = (torch.floor(torch.rand(n, 3, generator=g, device=dev, dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
    pos = pos[_ops.spatial_order(pos).long()].contiguous()
    feat = torch.randn(n, c, generator=g, device=dev)
    up = torch.randn(n, c, generator=g, device=dev)
    th = 0.1 * torch.randn(c, c, 3, generator=g, device=dev)
    tb = 0.1 * torch.randn(c, c, generator=g, device=dev)
    nbr = _ops.knn(pos, 1, n, k)
    csr = _ops.csr_build(nbr, 1, n)
    res = {"n": n, "k": k, "channels": f"{c}->{c}", "device": torch.cuda.get_device_name(0),
           "timing": "CUDA events, median of 5, per shard on its [owned | halo] buffers"}
    res["world_1"] = {"fwd_ms": round(timed(lambda: _ops.conv_forward(feat, pos, nbr, th, tb, 1, n)), 4),
                      "fwd_bwd_ms": round(timed(lambda: (_ops.conv_forward(feat, pos, nbr, th, tb, 1, n),
                                                         _ops.conv_backward(up, feat, pos, nbr, csr, th, tb, 1, n))), 4)}
    nbr_h = nbr.cpu().numpy()
    for world in (2, 4, 8):
        t0 = time.perf_counter()
        plans = parallel.HaloPlan.build_all(nbr_h, world)
        plan_s = time.perf_counter() - t0
        shards = []
        for p in plans:
            sel = torch.cat([torch.arange(p.lo, p.hi, device=dev), torch.from_numpy(p.halo).to(dev)])
            f_l, x_l, g_l = feat[sel].contiguous(), pos[sel].contiguous(), up[sel].contiguous()
            g_l[p.n_own:] = 0
            nb_l = torch.from_numpy(p.local_nbr).to(dev, torch.int32)
            m = p.n_local
            csr_l = _ops.csr_build(nb_l, 1, m)
            fwd = timed(lambda: _ops.conv_forward(f_l, x_l, nb_l, th, tb, 1, m))
            both = timed(lambda: (_ops.conv_forward(f_l, x_l, nb_l, th, tb, 1, m),
                                  _ops.conv_backward(g_l, f_l, x_l, nb_l, csr_l, th, tb, 1, m)))
            shards.append({"owned": p.n_own, "halo": int(len(p.halo)),
                           "halo_frac": round(len(p.halo) / p.n_own, 4),
                           "halo_recv_bytes_fwd": int(len(p.halo)) * (4 * c + 12),
                           "fwd_ms": round(fwd, 4), "fwd_bwd_ms": round(both, 4)})
            del f_l, x_l, g_l, nb_l, csr_l
        torch.cuda.empty_cache()
        worst = max(shards, key=lambda s: s["fwd_bwd_ms"])
        res[f"world_{world}"] = {
            "plan_build_s": round(plan_s, 2),
            "max_halo_frac": max(s["halo_frac"] for s in shards),
            "max_halo_recv_MB_fwd": round(max(s["halo_recv_bytes_fwd"] for s in shards) / 1e6, 2),
            "slowest_shard_fwd_ms": max(s["fwd_ms"] for s in shards),
            "slowest_shard_fwd_bwd_ms": worst["fwd_bwd_ms"],
            "compute_speedup_fwd_bwd": round(res["world_1"]["fwd_bwd_ms"] / worst["fwd_bwd_ms"], 2),
            "shards": shards,
        }
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

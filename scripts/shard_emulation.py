"""C4 (one 7M-point cloud, point-chunk sharded with halos) on ONE B200 by emulation: W ranks
(torchrun, gloo, all on cuda:0) run the product path -- parallel.ShardedCloud.build (sharded
exact kNN with the position ghost shell, device-resident halo plan) and ShardedFlexConv --
and then, one rank at a time (the others wait at a barrier, so each shard has the GPU to
itself), every rank times its own shard's kernels with CUDA events: the forward's interior
rows + boundary rows (fc_conv_forward_rows) and the backward, on its [owned | halo] buffers.
The halo exchange itself needs W GPUs (NVLink); its bytes are reported so its time can be
bounded.

  python -m torch.distributed.run --nproc-per-node W --master-addr 127.0.0.1 \\
      scripts/shard_emulation.py [--n 7000000]          (rank 0 prints one JSON object)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import torch
import torch.distributed as dist

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
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    n, k, c = args.n, args.k, args.c
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    pos = (torch.floor(torch.rand(n, 3, generator=g, device=dev, dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
    pos = pos[_ops.spatial_order(pos).long()].contiguous()
    lo, hi = parallel.shard_range(n, world, rank)
    feat = torch.randn(n, c, generator=g, device=dev)[lo:hi].contiguous()
    up = torch.randn(n, c, generator=g, device=dev)[lo:hi].contiguous()
    th = 0.1 * torch.randn(c, c, 3, generator=g, device=dev)
    tb = 0.1 * torch.randn(c, c, generator=g, device=dev)
    pos = pos[lo:hi].contiguous()
    torch.cuda.empty_cache()
    comm = parallel.Comm(device=dev)
    dist.barrier()
    t0 = time.perf_counter()
    cloud = parallel.ShardedCloud.build(pos, k, comm)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    f_l, g_l = cloud.local_buffer(feat), cloud.local_buffer(up)
    cloud.fill_halo(f_l)
    x_l = cloud.positions
    out = torch.empty(cloud.n_local, c, device=dev)
    stats = None
    for r in range(world):
        dist.barrier()
        if r == rank:
            fwd = timed(lambda: (_ops.conv_forward_rows(f_l, x_l, cloud.table, th, tb, cloud.interior_rows, out),
                                 _ops.conv_forward_rows(f_l, x_l, cloud.table, th, tb, cloud.boundary_rows, out)))
            bwd = timed(lambda: _ops.conv_backward(g_l, f_l, x_l, cloud.table, cloud.csr, th, tb, 1, cloud.n_local,
                                                   need=(True, True, True, True)))
            n_halo = cloud.n_local - cloud.n_own
            stats = [float(cloud.n_own), float(n_halo), float(cloud.n_ghost), float(cloud.interior_rows.numel()),
                     fwd, bwd, build_s, float(n_halo * (4 * c))]
        torch.cuda.synchronize()
    rows = [None] * world
    dist.all_gather_object(rows, stats)
    if rank == 0:
        shards = [{"owned": int(s[0]), "halo": int(s[1]), "halo_frac": round(s[1] / s[0], 4),
                   "ghost_frac": round(s[2] / s[0], 4), "interior_frac": round(s[3] / s[0], 4),
                   "fwd_ms": round(s[4], 4), "bwd_ms": round(s[5], 4), "fwd_bwd_ms": round(s[4] + s[5], 4),
                   "build_s": round(s[6], 2), "halo_recv_MB_fwd": round(s[7] / 1e6, 2)} for s in rows]
        worst = max(shards, key=lambda s: s["fwd_bwd_ms"])
        print(json.dumps({"n": n, "k": k, "channels": f"{c}->{c}", "world": world,
                          "device": torch.cuda.get_device_name(0),
                          "timing": "each shard alone on the GPU (the others wait at a barrier), CUDA events, "
                                    "median of 5; forward = interior rows + boundary rows (fc_conv_forward_rows)",
                          "slowest_shard_fwd_ms": max(s["fwd_ms"] for s in shards),
                          "slowest_shard_fwd_bwd_ms": worst["fwd_bwd_ms"],
                          "max_halo_frac": max(s["halo_frac"] for s in shards),
                          "max_ghost_frac": max(s["ghost_frac"] for s in shards),
                          "sharded_knn_and_plan_s_max": max(s["build_s"] for s in shards),
                          "shards": shards}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

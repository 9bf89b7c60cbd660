"""Where a U-Net training step's time goes (C5 shape, one 262,144-point scene): torch.profiler
table of device kernels and host ops, plus the library's own per-kernel event timer.

  python scripts/profile_c5.py [--n 262144] [--dtype f32|f64]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1803_07289_b200 import _lib, network, sampling  # noqa: E402
from paper_1803_07289_b200.core import PointCloud, Rng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=262_144)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--base", type=int, default=64)
    args = ap.parse_args()
    dt = torch.float32 if args.dtype == "f32" else torch.float64
    rng = np.random.default_rng(5)
    n = args.n
    loc = np.floor(rng.random((n, 3)) * 2 ** 24) / 2 ** 24
    feats = rng.standard_normal((n, 1))
    labels = rng.integers(0, 3, n)
    h = sampling.build_hierarchy(PointCloud(loc, feats), 8, 4, 2, Rng(5).spawn(1))
    g = network.build_segnet(3, 1, 3, 2, args.base, 8, 4, dtype=dt)
    network.initialize_params(g, Rng(5).spawn(2), h)
    adam = network.init_adam(g.store.size, lr=3e-3, dtype=dt)
    x = torch.from_numpy(feats).cuda().to(dt)
    lab = torch.from_numpy(labels).cuda()
    for _ in range(2):
        network.train_step(g, adam, h, x, lab)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        network.train_step(g, adam, h, x, lab)
    torch.cuda.synchronize()
    print(f"wall ms/step {(time.perf_counter() - t0) / 3 * 1e3:.2f}")
    with _lib.KernelTimer() as kt:
        network.train_step(g, adam, h, x, lab)
    for name, v in sorted(kt.times.items(), key=lambda kv: -sum(kv[1])):
        print(f"lib {name:24s} n={len(v):3d} total {sum(v):8.3f} ms")
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        network.train_step(g, adam, h, x, lab)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30))
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))


if __name__ == "__main__":
    main()

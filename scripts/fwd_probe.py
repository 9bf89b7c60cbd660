"""Forward-kernel timing probe (GPU box): time fc_conv_forward at the bench shape under
debug variants (FC_DBG bit flags read by the fast forward launcher) to locate the limiter.

    python scripts/fwd_probe.py [--n 7000000] [--variants 0,1,2,4]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=7_000_000)
    ap.add_argument("--variants", default="0")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--mode", default="auto")
    args = ap.parse_args()
    import torch

    from paper_1803_07289_b200 import _ops

    dev = torch.device("cuda")
    n, k, c, d = args.n, 8, 64, 3
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    pos = torch.floor(torch.rand(n, d, generator=gen, device=dev, dtype=torch.float64) * 2 ** 24) / 2 ** 24
    pos = pos.to(torch.float32)
    order = _ops.spatial_order(pos)
    pos = pos[order.long()].contiguous()
    feat = torch.randn(n, c, generator=gen, device=dev)
    theta = 0.1 * torch.randn(c, c, d, generator=gen, device=dev)
    theta_b = 0.1 * torch.randn(c, c, generator=gen, device=dev)
    nbr = _ops.knn(pos, 1, n, k)
    torch.cuda.synchronize()
    ref = None
    for v in args.variants.split(","):
        os.environ["FC_DBG"] = v
        for _ in range(3):
            out = _ops.conv_forward(feat, pos, nbr, theta, theta_b, 1, n, args.mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            out = _ops.conv_forward(feat, pos, nbr, theta, theta_b, 1, n, args.mode)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        if ref is None:
            ref = out.clone()
        diff = float((out - ref).abs().max())
        print(f"variant {v}: {ms:.3f} ms/fwd  {n / ms / 1e3:.1f} Mpts/s  {556 * n / ms / 1e6:.0f} GB/s(alg)  maxdiff-vs-first {diff:.3g}",
              flush=True)


if __name__ == "__main__":
    main()

"""Backward-kernel timing probe (GPU box): per-kernel times of fc_conv_backward at the bench
shape under FC_DBG variants (read by the fast kernels' launchers).

    python scripts/bwd_probe.py [--n 7000000] [--variants 0,2,8]
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
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    from paper_1803_07289_b200 import _lib, _ops

    dev = torch.device("cuda")
    n, k, c, d = args.n, 8, 64, 3
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    pos = torch.floor(torch.rand(n, d, generator=gen, device=dev, dtype=torch.float64) * 2 ** 24) / 2 ** 24
    pos = pos.to(torch.float32)
    order = _ops.spatial_order(pos)
    pos = pos[order.long()].contiguous()
    feat = torch.randn(n, c, generator=gen, device=dev)
    g = torch.randn(n, c, generator=gen, device=dev)
    theta = 0.1 * torch.randn(c, c, d, generator=gen, device=dev)
    theta_b = 0.1 * torch.randn(c, c, generator=gen, device=dev)
    nbr = _ops.knn(pos, 1, n, k)
    csr = _ops.csr_build(nbr, 1, n)
    torch.cuda.synchronize()
    ref = None
    for v in args.variants.split(","):
        os.environ["FC_DBG"] = v
        for _ in range(2):
            _ops.conv_backward(g, feat, pos, nbr, csr, theta, theta_b, 1, n, need=(True, True, True, True))
        torch.cuda.synchronize()
        with _lib.KernelTimer() as kt:
            for _ in range(args.reps):
                out = _ops.conv_backward(g, feat, pos, nbr, csr, theta, theta_b, 1, n, need=(True, True, True, True))
            torch.cuda.synchronize()
        if ref is None:
            ref = [x.clone() for x in out]
        diff = max(float((a - b).abs().max()) for a, b in zip(out, ref))
        ms = {name: sum(t) / len(t) for name, t in kt.times.items()}
        print(f"variant {v}: " + "  ".join(f"{name} {m:.3f} ms" for name, m in sorted(ms.items())) + f"  maxdiff {diff:.3g}",
              flush=True)


if __name__ == "__main__":
    main()

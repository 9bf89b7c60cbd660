"""Host<->device copy bandwidth probe (GPU box): pinned H2D alone, D2H alone, and both at
once on two streams -- the bound on bench.py's e2e leg (inputs H2D + results D2H per step).

    python scripts/pcie_probe.py [--mb 1024]
"""
import argparse


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    nb = args.mb << 20
    h_src = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.reps / 1e3

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(f"H2D {nb / t1 / 1e9:.1f} GB/s  D2H {nb / t2 / 1e9:.1f} GB/s  both {2 * nb / t3 / 1e9:.1f} GB/s "
          f"({nb / t3 / 1e9:.1f} each way)")


if __name__ == "__main__":
    main()

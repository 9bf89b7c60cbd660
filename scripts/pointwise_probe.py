"""Pointwise-GEMM timing on the C5 U-Net's shapes: the tcgen05 kernel (fc_gemm_rows /
fc_gemm_wgrad) against torch/cuBLAS SGEMM for the same products (CUDA events, median of 20).
   python scripts/pointwise_probe.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_07289_b200 import _ops  # noqa: E402


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


SHAPES = [(262144, [64, 3], 64), (262144, [128, 64, 3], 64), (65536, [128, 3], 128), (65536, [256, 128, 3], 128),
          (16384, [256, 3], 256), (262144, [64], 3)]
dev = torch.device("cuda", 0)
for n, widths, co in SHAPES:
    xs = [torch.randn(n, w, device=dev) for w in widths]
    ci = sum(widths)
    w = torch.randn(co, ci, device=dev)
    b = torch.randn(co, device=dev)
    g = torch.randn(n, co, device=dev)
    segs, a0 = [], 0
    for wd in widths:
        segs.append((a0, wd))
        a0 += wd
    img = _ops.gemm_pack(w, segs)
    imgt = _ops.gemm_pack(w, [(0, co)], transpose=True)
    dw, db = torch.empty(co, ci, device=dev), torch.empty(co, device=dev)
    fwd = t(lambda: _ops.gemm_rows(xs, img, co, bias=b, relu=True))
    dgr = t(lambda: _ops.gemm_rows([g], imgt, ci, outs=[(s, s + wd) for s, wd in segs]))
    wgr = t(lambda: _ops.gemm_wgrad(g, xs, dw, db))

    def tf():
        y = None
        for x, (s, wd) in zip(xs, segs):
            y = torch.addmm(b, x, w[:, s:s + wd].t()) if y is None else y.addmm_(x, w[:, s:s + wd].t())
        return y, torch.clamp_min(y, 0)

    def td():
        return [g @ w[:, s:s + wd] for s, wd in segs]

    def tw():
        for x, (s, wd) in zip(xs, segs):
            dw[:, s:s + wd] = g.t() @ x
        torch.sum(g, 0, out=db)
    print(f"n={n} {widths}->{co}: fwd {fwd:.3f} (cublas {t(tf):.3f}) dgrad {dgr:.3f} (cublas {t(td):.3f}) "
          f"wgrad {wgr:.3f} (cublas {t(tw):.3f}) ms")

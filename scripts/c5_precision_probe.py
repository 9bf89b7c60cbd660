"""C5 architecture (base_channels=64) fp32 step vs the reference golden: error budget of the
fp32 engines, with the pointwise GEMMs on the tcgen05 kernel (default) or on torch/cuBLAS
(--torch-pointwise) for comparison.   python scripts/c5_precision_probe.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1803_07289_b200 import network, sampling  # noqa: E402
from paper_1803_07289_b200.core import PointCloud, Rng  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def run(seg, torch_pw):
    if torch_pw:
        orig_dtype = network.ParamStore.__init__

        class _Fake(torch.dtype.__class__):
            pass
        # route the fp32 pointwise GEMMs through torch by making the dtype test fail
        fwd, bwd = network._MultiGemm.forward, network._MultiGemm.backward

        def f(self, ops, relu=False):
            w, b = self.store.view(self.name + ".w"), self.store.view(self.name + ".b")
            y = None
            for label, a, c in self.cols():
                y = torch.addmm(b, ops[label], w[:, a:c].t()) if y is None else y.addmm_(ops[label], w[:, a:c].t())
            return (y, torch.clamp_min(y, 0)) if relu else y

        def bk(self, g, ops, grads, need=(), mask=None):
            w = self.store.view(self.name + ".w")
            gw, gb = self.store.view(self.name + ".w", grads), self.store.view(self.name + ".b", grads)
            if mask is not None:
                g = g * (mask > 0)
            torch.sum(g, dim=0, out=gb)
            out = {}
            for label, a, c in self.cols():
                gw[:, a:c] = g.t() @ ops[label]
                if label in need:
                    out[label] = g @ w[:, a:c]
            return out
        network._MultiGemm.forward, network._MultiGemm.backward = f, bk
    cloud = PointCloud(seg["locations"], seg["features"])
    h = sampling.build_hierarchy(cloud, 8, 4, 2, Rng(7).spawn(1))
    g = network.build_segnet(3, 1, 3, 2, 64, 8, 4, dtype=torch.float32)
    network.initialize_params(g, Rng(7).spawn(2), h)
    logits = g.forward(h, cloud.features)
    loss, lg = network.softmax_cross_entropy(logits, seg["labels"])
    grads = g.backward(lg)
    names = list(seg["param_names"])
    norms = np.array([float(torch.linalg.norm(g.store.view(nm, torch.from_numpy(grads)).double())) for nm in names])
    nz = seg["grad_norms"] > 0
    pl = np.abs(norms[nz] - seg["grad_norms"][nz]) / seg["grad_norms"][nz]
    s = grads[seg["grad_idx"]]
    ref = seg["grad_sample"]
    print({"pointwise": "torch" if torch_pw else "tcgen05", "logits_rel": rel(logits, seg["logits"]),
           "loss_rel": abs(loss - float(seg["loss"])) / abs(float(seg["loss"])),
           "grad_norm_rel": abs(np.linalg.norm(grads) - float(seg["grad_norm"])) / float(seg["grad_norm"]),
           "per_layer_norm_rel_max": float(pl.max()), "sample_rel": rel(s, ref),
           "sample_max_abs_over_max": float(np.abs(s - ref).max() / np.abs(ref).max())})


seg = dict(np.load(os.path.join(ROOT, "tests", "golden", "network_segnet64.npz")))
run(seg, "--torch-pointwise" in sys.argv)

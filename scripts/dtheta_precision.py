"""d_theta / d_theta_b precision of the fp32 engines against the full fp64 oracle reduction,
as a function of the cloud size (the tensor-core engine accumulates each CTA's share of the
points in TMEM; the SIMT engine reduces fp32 partials in fp64).
    python scripts/dtheta_precision.py [--sizes 20000,100000,...]  -> JSON lines"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_1803_07289_b200 import _ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="20000,100000,300000,1048576,3000000")
    ap.add_argument("--modes", default="split,simt")
    args = ap.parse_args()
    import bench

    for n in [int(x) for x in args.sizes.split(",")]:
        w = bench.make_workload(n, 8, 64, 0, torch.device("cuda", 0))
        h = {k: w[k].cpu().numpy().astype(np.float64) for k in ("pos", "feat", "g")}
        nbr = w["nbr"].cpu().numpy().astype(np.int64)
        rth, rtb = oracle.conv_param_grads(h["g"], h["feat"], h["pos"], nbr)
        for mode in args.modes.split(","):
            _, dth, dtb, _ = _ops.conv_backward(w["g"], w["feat"], w["pos"], w["nbr"], None, w["theta"], w["theta_b"],
                                                1, n, need=(False, True, True, False), mode=mode)
            out = {"n": n, "mode": mode}
            for name, got, ref in (("d_theta", dth, rth), ("d_theta_b", dtb, rtb)):
                got = got.cpu().numpy().astype(np.float64)
                err = got - ref
                out[name] = {"norm_rel": float(np.linalg.norm(err) / np.linalg.norm(ref)),
                             "max_abs": float(np.abs(err).max()), "max_ref": float(np.abs(ref).max()),
                             "mean_signed_rel": float((err * np.sign(ref)).sum() / np.abs(ref).sum())}
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

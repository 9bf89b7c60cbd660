"""Worker for tests/test_gpu_parallel.py: point-chunk sharding on the GPU with the product
kernels (libflexconv_b200.so) -- several ranks on the one GPU of the test box, gloo
transport (host staging).  Compares with the unsharded CUDA operator on the whole cloud."""

import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1803_07289_b200 import _ops, parallel  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    n, k, c = int(os.environ.get("FC_SHARD_N", "200000")), 8, 64
    gen = torch.Generator(device=dev)
    gen.manual_seed(77)  # identical cloud on every rank (each keeps only its block)
    pos = (torch.floor(torch.rand(n, 3, generator=gen, device=dev, dtype=torch.float64) * 2 ** 24) / 2 ** 24).float()
    pos[n - 500:] = pos[1000:1500]  # duplicates far apart in index: global tie-breaking
    pos = pos[_ops.spatial_order(pos).long()].contiguous()
    feat = torch.randn(n, c, generator=gen, device=dev)
    g = torch.randn(n, c, generator=gen, device=dev)
    th = 0.1 * torch.randn(c, c, 3, generator=gen, device=dev)
    tb = 0.1 * torch.randn(c, c, generator=gen, device=dev)
    lo, hi = parallel.shard_range(n, world, rank)

    comm = parallel.Comm(device=dev)
    cloud = parallel.ShardedCloud.build(pos[lo:hi], k, comm)
    layer = parallel.ShardedFlexConv(cloud)
    out = layer.forward(feat[lo:hi], th, tb)
    df, dth, dtb, dl = layer.backward(g[lo:hi])

    nbr = _ops.knn(pos, 1, n, k)
    csr = _ops.csr_build(nbr, 1, n)
    ref_out = _ops.conv_forward(feat, pos, nbr, th, tb, 1, n)
    rdf, rdth, rdtb, rdl = _ops.conv_backward(g, feat, pos, nbr, csr, th, tb, 1, n)

    def rel(a, b):
        return float((a.double() - b.double()).abs().max() / b.double().abs().max())

    res = {"rank": rank, "halo": int(cloud.halo.numel()), "ghosts": cloud.n_ghost,
           "halo_fraction": cloud.halo_fraction,
           "knn_rows_exact": bool(torch.equal(cloud.global_rows, nbr[lo:hi].long())),
           "fwd_bitwise": bool(torch.equal(out, ref_out[lo:hi])),
           "df_err": rel(df, rdf[lo:hi]), "dl_err": rel(dl, rdl[lo:hi]),
           "dth_err": rel(dth, rdth), "dtb_err": rel(dtb, rdtb)}
    with open(os.path.join(os.environ["FC_RESULT_DIR"], f"rank{rank}.json"), "w") as fh:
        json.dump(res, fh)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Worker for tests/test_parallel.py: launched with torch.distributed.run (gloo, CPU).

Point-chunk sharding of one cloud (parallel.ShardedCloud / ShardedFlexConv): every rank
holds only its block of the spatially ordered cloud; the sharded kNN (ghost shell), the
halo plan, the halo exchanges and the gradient reductions under test are product code.
The per-rank arithmetic (kNN, flex-conv forward / backward) is the CPU ORACLE here (test
infrastructure) because this host has no GPU; tests/test_gpu_parallel.py runs the same
path with the CUDA kernels.  Also checks the batch-sharded gradient combination.
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_1803_07289_b200 import parallel  # noqa: E402
from paper_1803_07289_b200.core import synthetic_layer  # noqa: E402


def oracle_kernels():
    def knn(points, k):
        return torch.from_numpy(oracle.knn_brute(points.numpy().astype(np.float64), k))

    def conv_fwd(feat, loc, nbr, th, tb):
        return torch.from_numpy(oracle.conv_forward(feat.numpy(), loc.numpy(), nbr.numpy(), th.numpy(), tb.numpy(), 1))

    def conv_bwd(g, feat, loc, nbr, csr, th, tb, need):
        out = oracle.conv_backward(g.numpy(), feat.numpy(), loc.numpy(), nbr.numpy(), th.numpy(), tb.numpy())
        return tuple(torch.from_numpy(x) for x in out)

    def conv_fwd_rows(feat, loc, nbr, th, tb, rows, out):
        # the rows from the CURRENT feature buffer: rows computed before the halo exchange
        # completed (the interior rows) are wrong if they touch a halo row
        full = oracle.conv_forward(feat.numpy(), loc.numpy(), nbr.numpy(), th.numpy(), tb.numpy(), 1)
        r = rows.long()
        out[r] = torch.from_numpy(full)[r]
        return out

    return {"knn": knn, "conv_fwd": conv_fwd, "conv_bwd": conv_bwd, "csr": lambda nbr: None,
            "conv_fwd_rows": conv_fwd_rows}


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    n, k, cin, cout = 3000, 8, 6, 5
    loc, feat, th, tb, up = synthetic_layer(41, 0, n, 3, cin, cout)
    # exact duplicates across the cloud (index tie-breaking must be the global one)
    loc[2500:2520] = loc[10:30]
    # spatial order (x-major sort is enough for a test), identical on all ranks
    order = np.lexsort((loc[:, 2], loc[:, 1], loc[:, 0]))
    loc, feat, up = loc[order], feat[order], up[order]
    lo, hi = parallel.shard_range(n, world, rank)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    comm = parallel.Comm(device=torch.device("cpu"))
    cloud = parallel.ShardedCloud.build(t(loc[lo:hi]), k, comm, kernels=oracle_kernels())
    ref_nbr = oracle.knn_brute(loc, k)
    layer = parallel.ShardedFlexConv(cloud)
    out = layer.forward(t(feat[lo:hi]), t(th), t(tb))
    df, dth, dtb, dl = layer.backward(t(up[lo:hi]))
    ref_out = oracle.conv_forward(feat, loc, ref_nbr, th, tb, 1)
    rdf, rdth, rdtb, rdl = oracle.conv_backward(up, feat, loc, ref_nbr, th, tb)
    res = {
        "rank": rank,
        "bounds": cloud.bounds,
        "halo": int(cloud.halo.numel()),
        "ghosts": cloud.n_ghost,
        "knn_rows_exact": bool(np.array_equal(cloud.global_rows.numpy(), ref_nbr[lo:hi])),
        "halo_outside": bool(((cloud.halo < lo) | (cloud.halo >= hi)).all()),
        "interior_boundary_partition": bool(cloud.interior_rows.numel() + cloud.boundary_rows.numel() == hi - lo
                                            and cloud.boundary_rows.numel() > 0 and cloud.interior_rows.numel() > 0),
        "fwd_bitwise": bool(np.array_equal(out.numpy(), ref_out[lo:hi])),
        "df_err": float(np.abs(df.numpy() - rdf[lo:hi]).max() / np.abs(rdf).max()),
        "dl_err": float(np.abs(dl.numpy() - rdl[lo:hi]).max() / np.abs(rdl).max()),
        "dth_err": float(np.abs(dth.numpy() - rdth).max() / np.abs(rdth).max()),
        "dtb_err": float(np.abs(dtb.numpy() - rdtb).max() / np.abs(rdtb).max()),
    }
    # determinism of the whole sharded backward (fixed-order reductions)
    layer.forward(t(feat[lo:hi]), t(th), t(tb))
    again = layer.backward(t(up[lo:hi]))
    res["backward_bitwise_repeat"] = bool(all(torch.equal(a, b) for a, b in zip(again, (df, dth, dtb, dl))))
    # batch-sharded gradient combination (network.train_step_batch): per-unit rows summed in
    # global unit order must equal the single-process sequential loop bitwise
    units = 5
    rows = torch.from_numpy(np.random.default_rng(7).standard_normal((units, 33)) * 10.0 ** np.arange(-8, 25, 1))
    lo_u, hi_u = parallel.shard_range(units, world, rank)
    got = parallel.ordered_allgather_sum(rows[lo_u:hi_u].clone(), units)
    seq = torch.zeros(33, dtype=torch.float64)
    for r in rows:
        seq += r
    res["ordered_sum_bitwise"] = bool(torch.equal(got, seq))
    out_dir = os.environ.get("FC_RESULT_DIR")
    if out_dir:  # one file per rank: the ranks' stdout lines can interleave
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
            json.dump(res, fh)
    else:
        print("RESULT " + json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

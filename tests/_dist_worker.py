"""Worker for tests/test_parallel.py: launched with torch.distributed.run (gloo, CPU).

Checks that point-chunk sharding with halos (paper_1803_07289_b200.parallel) reproduces
the unsharded flex-conv forward / backward.  The compute callback here is the CPU ORACLE
(test infrastructure): the sharding, halo exchange and reductions under test are product
code; only the per-shard arithmetic is stood in for, because this host has no GPU.
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


def oracle_compute():
    def fwd(feat, loc, nbr, th, tb):
        return torch.from_numpy(oracle.conv_forward(feat.numpy(), loc.numpy(), nbr, th.numpy(), tb.numpy(), 1))

    def bwd(g, feat, loc, nbr, th, tb):
        df, dth, dtb, dl = oracle.conv_backward(g.numpy(), feat.numpy(), loc.numpy(), nbr, th.numpy(), tb.numpy())
        return tuple(torch.from_numpy(x) for x in (df, dth, dtb, dl))

    return fwd, bwd


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    n, k, cin, cout = 3000, 8, 6, 5
    loc, feat, th, tb, up = synthetic_layer(41, 0, n, 3, cin, cout)
    # spatial order (x-major sort is enough for a test) + exact kNN, identical on all ranks
    order = np.lexsort((loc[:, 2], loc[:, 1], loc[:, 0]))
    loc, feat, up = loc[order], feat[order], up[order]
    nbr = oracle.knn_brute(loc, k)
    tr = parallel.DistTransport()
    plan = parallel.HaloPlan.build_local(nbr, world, rank, tr)
    ref_plan = parallel.HaloPlan.build_all(nbr, world)[rank]
    same_plan = (np.array_equal(plan.halo, ref_plan.halo) and np.array_equal(plan.local_nbr, ref_plan.local_nbr)
                 and sorted(plan.send_lists) == sorted(ref_plan.send_lists)
                 and all(np.array_equal(plan.send_lists[d], ref_plan.send_lists[d]) for d in plan.send_lists))
    lo, hi = plan.lo, plan.hi
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    feat_l = plan.gather_halo(t(feat[lo:hi]), tr)
    loc_l = plan.gather_halo(t(loc[lo:hi]), tr)
    comp = oracle_compute()
    out = parallel.sharded_forward(plan, feat_l, loc_l, t(th), t(tb), comp)
    df_l, dth, dtb, dl_l = parallel.sharded_backward_local(plan, t(up[lo:hi]), feat_l, loc_l, t(th), t(tb), comp)
    df = plan.scatter_halo_add(df_l, tr)
    dl = plan.scatter_halo_add(dl_l, tr)
    dth = parallel.fixed_order_allreduce(dth)
    dtb = parallel.fixed_order_allreduce(dtb)
    # unsharded reference
    ref_out = oracle.conv_forward(feat, loc, nbr, th, tb, 1)
    rdf, rdth, rdtb, rdl = oracle.conv_backward(up, feat, loc, nbr, th, tb)
    res = {
        "rank": rank,
        "halo": int(len(plan.halo)),
        "same_plan": bool(same_plan),
        "fwd_bitwise": bool(np.array_equal(out.numpy(), ref_out[lo:hi])),
        "df_err": float(np.abs(df.numpy() - rdf[lo:hi]).max() / np.abs(rdf).max()),
        "dl_err": float(np.abs(dl.numpy() - rdl[lo:hi]).max() / np.abs(rdl).max()),
        "dth_err": float(np.abs(dth.numpy() - rdth).max() / np.abs(rdth).max()),
        "dtb_err": float(np.abs(dtb.numpy() - rdtb).max() / np.abs(rdtb).max()),
    }
    # determinism of the fixed-order reduction
    again = parallel.fixed_order_allreduce(parallel.sharded_backward_local(
        plan, t(up[lo:hi]), feat_l, loc_l, t(th), t(tb), comp)[1])
    res["allreduce_bitwise"] = bool(torch.equal(again, dth))
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
    if out_dir:  # one file per rank: the two ranks' stdout lines can interleave
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
            json.dump(res, fh)
    else:
        print("RESULT " + json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

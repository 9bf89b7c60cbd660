"""CPU, multi-process (gloo, world_size 2): batch sharding and point-chunk sharding with
halos reproduce the unsharded operator (tests/_dist_worker.py)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    from paper_1803_07289_b200.parallel import shard_range

    for units in (0, 1, 7, 32, 1000):
        for world in (1, 2, 3, 8):
            got = [shard_range(units, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == units
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [h - lo for lo, h in got]
            assert max(sizes) - min(sizes) <= 1


def test_halo_plan_invariants(oracle_mod):
    from paper_1803_07289_b200.parallel import HaloPlan
    from paper_1803_07289_b200.core import Rng, lattice_positions

    pts = lattice_positions(Rng(5).gen, 2000, 3)
    pts = pts[np.lexsort((pts[:, 2], pts[:, 1], pts[:, 0]))]
    nbr = oracle_mod.knn_brute(pts, 8)
    plans = HaloPlan.build_all(nbr, 3)
    for p in plans:
        assert p.local_nbr.shape == (p.n_local, 8)
        # remapped rows point at the same global points
        glob = np.concatenate([np.arange(p.lo, p.hi), p.halo])
        np.testing.assert_array_equal(glob[p.local_nbr[: p.n_own]], nbr[p.lo:p.hi])
        assert not np.isin(p.halo, np.arange(p.lo, p.hi)).any()
        for src, pos in p.recv_lists.items():
            np.testing.assert_array_equal(plans[src].send_lists[p.rank] + plans[src].lo, p.halo[pos])


@pytest.mark.timeout(300)
def test_point_chunk_sharding_gloo_world2(oracle_mod, tmp_path):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1", FC_RESULT_DIR=str(tmp_path))
    for attempt in range(3):  # retries only guard against a rendezvous-port race
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.join(ROOT, "tests", "_dist_worker.py")]
        proc = subprocess.run(cmd, capture_output=True, text=True, timeout=140, env=env, cwd=ROOT)
        if proc.returncode == 0:
            break
    assert proc.returncode == 0, proc.stderr[-3000:]
    res = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(2)]
    assert len(res) == 2
    for r in res:
        assert r["halo"] > 0
        assert r["same_plan"]
        assert r["fwd_bitwise"]
        assert r["df_err"] < 1e-12 and r["dl_err"] < 1e-12
        assert r["dth_err"] < 1e-12 and r["dtb_err"] < 1e-12
        assert r["allreduce_bitwise"]
        assert r["ordered_sum_bitwise"]

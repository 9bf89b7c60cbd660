"""GPU: point-chunk sharding of one cloud (parallel.ShardedCloud / ShardedFlexConv) with
the product kernels, 2 and 4 ranks sharing the test box's GPU (gloo transport), against
the unsharded CUDA operator: ghost-shell kNN rows exact, forward rows bitwise, backward to
fp32 rounding (the owners add the other ranks' halo partials after their own sums)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_point_chunk_sharding_on_gpu(fc, tmp_path, world):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1", FC_RESULT_DIR=str(tmp_path))
    for attempt in range(3):  # retries only guard against a rendezvous-port race
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.join(ROOT, "tests", "_dist_worker_gpu.py")]
        proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
        if proc.returncode == 0:
            break
    assert proc.returncode == 0, proc.stderr[-4000:]
    for r in range(world):
        res = json.loads((tmp_path / f"rank{r}.json").read_text())
        assert res["halo"] > 0 and res["ghosts"] >= res["halo"], res
        assert res["knn_rows_exact"], res
        assert res["fwd_bitwise"], res
        assert res["df_err"] < 1e-5 and res["dl_err"] < 1e-5, res
        assert res["dth_err"] < 1e-5 and res["dtb_err"] < 1e-5, res

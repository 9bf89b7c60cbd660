"""Multi-GPU sharding of the flex-convolution hot path.

The reference is single-process (its only parallelism is OpenMP over points and a Python
loop over clouds with gradient accumulation, harness.py:589-599).  Two partitionings:

* Batch sharding (configs C2 / C5): clouds are independent units; rank r takes a
  contiguous block of clouds (`shard_range`).  The only collective is the theta / theta_b
  gradient sum of the training step, done by `fixed_order_allreduce`: all-gather, then sum
  in rank order in fp64 -- bitwise reproducible for a given world size (no float
  reduction-order nondeterminism).

* Point-chunk sharding of ONE large cloud with neighbour halos (config C4, 7M points):
  after a spatial ordering the cloud is cut into contiguous row ranges; `HaloPlan` computes,
  once per neighbourhood, the halo (neighbours owned elsewhere), the grouped point-to-point
  exchange lists and the local neighbour table.  Forward = halo gather + local flex_conv.
  Backward = local backward with zero upstream on halo rows, then the halo rows' partial
  d_features / d_locations are sent back to their owners and added in fixed rank order, and
  d_theta / d_theta_b are summed with `fixed_order_allreduce`.  Results equal the
  unsharded operator (tests/test_parallel.py checks this against the oracle with gloo).

Transport: `DistTransport` (torch.distributed grouped isend/irecv -- NCCL over NVLink on
the GPU box, gloo for the CPU tests; gloo has no all-to-all) or `LocalTransport` (all ranks
in one process, used to emulate a sharded run on one GPU).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import ConfigInvalidError, ShapeMismatchError


# ---------------------------------------------------------------------------- batch sharding
def shard_range(units: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of `units` owned by `rank` (first ranks take the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigInvalidError(f"bad rank {rank} for world {world}")
    base, rem = divmod(units, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def fixed_order_allreduce(t: torch.Tensor, group=None) -> torch.Tensor:
    """Sum of `t` over ranks, accumulated in rank order in fp64 (deterministic)."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return t
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t.contiguous(), group=group)
    acc = torch.zeros_like(t, dtype=torch.float64)
    for p in parts:
        acc += p.to(torch.float64)
    return acc.to(t.dtype)


def ordered_allgather_sum(local: torch.Tensor, units: int, group=None) -> torch.Tensor:
    """Sum of per-unit rows in GLOBAL unit order, whatever the world size.

    `local` is [n_local, ...]: this rank's units, the block `shard_range(units, world, rank)`.
    Every rank all-gathers the blocks (padded to the largest) and adds the rows one by one in
    unit order, in `local`'s dtype -- the additions of the reference's sequential
    accumulation loop (harness.py:589-595: grads += graph.backward(g) per scene), so the
    result is bitwise identical for 1, 2, 4 or 8 ranks and to the single-process loop."""
    import torch.distributed as dist

    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    world = dist.get_world_size(group) if multi else 1
    rank = dist.get_rank(group) if multi else 0
    lo, hi = shard_range(units, world, rank)
    if local.shape[0] != hi - lo:
        raise ShapeMismatchError(f"rank {rank} holds {local.shape[0]} units, its shard is {hi - lo}")
    if not multi:
        blocks = [local]
    else:
        width = shard_range(units, world, 0)[1]  # the first block is the largest
        pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        blocks = [parts[r][: shard_range(units, world, r)[1] - shard_range(units, world, r)[0]]
                  for r in range(world)]
    acc = torch.zeros(tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    for b in blocks:
        for row in b:
            acc += row
    return acc


# ---------------------------------------------------------------------------- transports
class DistTransport:
    """Grouped point-to-point exchange over torch.distributed (one call per direction)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange(self, sends: dict, recv_shapes: dict, dtype, device) -> dict:
        """sends[r] -> tensor to rank r; returns {r: tensor received from r}."""
        ops, recvs = [], {}
        for r, shape in recv_shapes.items():
            buf = torch.empty(shape, dtype=dtype, device=device)
            recvs[r] = buf
            ops.append(self.dist.P2POp(self.dist.irecv, buf, r, self.group))
        for r, t in sends.items():
            ops.append(self.dist.P2POp(self.dist.isend, t.contiguous(), r, self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        return recvs


class LocalTransport:
    """All ranks live in this process (sequential emulation of a sharded run)."""

    def __init__(self, world: int):
        self.world = world
        self.mailbox: dict = {}

    def post(self, src: int, sends: dict):
        for dst, t in sends.items():
            self.mailbox[(src, dst)] = t

    def collect(self, dst: int, srcs) -> dict:
        return {s: self.mailbox.pop((s, dst)) for s in srcs}


# ---------------------------------------------------------------------------- halo plan
@dataclass
class HaloPlan:
    """Rank `rank`'s view of a point-chunk sharded cloud.

    owned rows [lo, hi) of the global (spatially ordered) point set; `halo` = sorted global
    ids of neighbours owned elsewhere; local point ids: owned j -> j - lo, halo[q] ->
    n_own + q.  `local_nbr` is [n_own + n_halo, K] (halo rows are self-loops: they carry
    zero upstream gradient and their forward outputs are discarded).
    """

    rank: int
    world: int
    lo: int
    hi: int
    halo: np.ndarray                # [n_halo] global ids
    recv_lists: dict                # src rank -> positions in `halo` (ascending)
    send_lists: dict                # dst rank -> owned local ids requested by dst
    local_nbr: np.ndarray           # [n_own + n_halo, K] int64

    @property
    def n_own(self) -> int:
        return self.hi - self.lo

    @property
    def n_local(self) -> int:
        return self.n_own + len(self.halo)

    @staticmethod
    def bounds(n: int, world: int) -> list[int]:
        return [shard_range(n, world, r)[0] for r in range(world)] + [n]

    @staticmethod
    def requests(nbr: np.ndarray, bounds: list[int], rank: int):
        """Halo ids of `rank` and, per owner, the positions in the halo they fill."""
        lo, hi = bounds[rank], bounds[rank + 1]
        rows = np.asarray(nbr[lo:hi], dtype=np.int64)
        if rows.size and (rows.min() < 0 or rows.max() >= bounds[-1]):
            raise ShapeMismatchError("neighbour index out of the sharded point range")
        ext = rows[(rows < lo) | (rows >= hi)]
        halo = np.unique(ext)
        owner = np.searchsorted(np.asarray(bounds), halo, side="right") - 1
        recv = {int(r): np.nonzero(owner == r)[0] for r in np.unique(owner)}
        return halo, recv

    @classmethod
    def build_all(cls, nbr, world: int, bounds: list[int] | None = None) -> list["HaloPlan"]:
        """Plans of every rank from the full neighbour table (host-side, once per
        neighbourhood; each rank can also build only its own with `build_local`)."""
        nbr = np.asarray(nbr, dtype=np.int64)
        n = nbr.shape[0]
        bounds = bounds or cls.bounds(n, world)
        reqs = [cls.requests(nbr, bounds, r) for r in range(world)]
        plans = []
        for r in range(world):
            halo, recv = reqs[r]
            send = {}
            for d in range(world):
                if d == r:
                    continue
                h_d, rv_d = reqs[d]
                if r in rv_d:
                    send[d] = h_d[rv_d[r]] - bounds[r]
            plans.append(cls._finish(r, world, bounds, nbr, halo, recv, send))
        return plans

    @classmethod
    def build_local(cls, nbr, world: int, rank: int, transport: DistTransport,
                    bounds: list[int] | None = None) -> "HaloPlan":
        """This rank's plan; request lists are exchanged with the owners (p2p)."""
        nbr = np.asarray(nbr, dtype=np.int64)
        n = nbr.shape[0]
        bounds = bounds or cls.bounds(n, world)
        halo, recv = cls.requests(nbr, bounds, rank)
        # 1) counts to every other rank, 2) the id lists
        counts = {d: torch.tensor([len(recv.get(d, []))], dtype=torch.int64) for d in range(world) if d != rank}
        got = transport.exchange(counts, {d: (1,) for d in counts}, torch.int64, torch.device("cpu"))
        sends = {d: torch.from_numpy(halo[recv[d]]) for d in recv}
        shapes = {d: (int(c.item()),) for d, c in got.items() if int(c.item()) > 0}
        ids = transport.exchange(sends, shapes, torch.int64, torch.device("cpu"))
        send = {d: t.numpy() - bounds[rank] for d, t in ids.items()}
        return cls._finish(rank, world, bounds, nbr, halo, recv, send)

    @classmethod
    def _finish(cls, rank, world, bounds, nbr, halo, recv, send) -> "HaloPlan":
        lo, hi = bounds[rank], bounds[rank + 1]
        rows = np.asarray(nbr[lo:hi], dtype=np.int64)
        n_own = hi - lo
        remap = np.empty(rows.shape, dtype=np.int64)
        inside = (rows >= lo) & (rows < hi)
        remap[inside] = rows[inside] - lo
        remap[~inside] = n_own + np.searchsorted(halo, rows[~inside])
        k = rows.shape[1] if rows.ndim == 2 else nbr.shape[1]
        halo_rows = np.repeat((n_own + np.arange(len(halo), dtype=np.int64))[:, None], k, axis=1)
        local = np.concatenate([remap, halo_rows], axis=0) if len(halo) else remap
        return cls(rank, world, lo, hi, halo, {int(r): v for r, v in recv.items()},
                   {int(d): np.asarray(v, dtype=np.int64) for d, v in send.items()}, local)

    # ------------------------------------------------------------------ exchanges
    def _send_rows(self, owned: torch.Tensor) -> dict:
        return {d: owned[torch.as_tensor(ids, device=owned.device)] for d, ids in self.send_lists.items()}

    def gather_halo(self, owned: torch.Tensor, transport) -> torch.Tensor:
        """[n_own, C] owned rows -> [n_own + n_halo, C] with the halo rows filled in."""
        c = owned.shape[1:]
        out = torch.empty((self.n_local,) + tuple(c), dtype=owned.dtype, device=owned.device)
        out[: self.n_own] = owned
        if isinstance(transport, DistTransport):
            got = transport.exchange(self._send_rows(owned),
                                     {s: (len(p),) + tuple(c) for s, p in self.recv_lists.items()},
                                     owned.dtype, owned.device)
        else:
            got = transport.collect(self.rank, self.recv_lists.keys())
        for s, pos in self.recv_lists.items():
            out[self.n_own + torch.as_tensor(pos, device=owned.device)] = got[s].to(owned.device)
        return out

    def post_halo(self, owned: torch.Tensor, transport: LocalTransport):
        """LocalTransport only: publish this rank's rows for the others' gather_halo."""
        transport.post(self.rank, self._send_rows(owned))

    def _halo_partials(self, local: torch.Tensor) -> dict:
        return {s: local[self.n_own + torch.as_tensor(pos, device=local.device)] for s, pos in self.recv_lists.items()}

    def scatter_halo_add(self, local: torch.Tensor, transport) -> torch.Tensor:
        """Return the owned rows of `local` plus every other rank's partial contribution
        to them, added in ascending source-rank order (deterministic)."""
        c = local.shape[1:]
        owned = local[: self.n_own].clone()
        if isinstance(transport, DistTransport):
            got = transport.exchange(self._halo_partials(local),
                                     {d: (len(ids),) + tuple(c) for d, ids in self.send_lists.items()},
                                     local.dtype, local.device)
        else:
            got = transport.collect(self.rank, self.send_lists.keys())
        for d in sorted(got):
            idx = torch.as_tensor(self.send_lists[d], device=local.device)
            owned.index_add_(0, idx, got[d].to(local.device))  # ids unique per source
        return owned

    def post_partials(self, local: torch.Tensor, transport: LocalTransport):
        transport.post(self.rank, self._halo_partials(local))


# ---------------------------------------------------------------------------- sharded layer
def cuda_compute():
    """The product compute: flex-conv forward / backward through libflexconv_b200.so."""
    from . import _ops

    def fwd(feat, loc, nbr, theta, theta_b):
        nbr32 = torch.as_tensor(nbr).to(feat.device, torch.int32)
        return _ops.conv_forward(feat, loc, nbr32, theta, theta_b, 1, feat.shape[0])

    def bwd(g, feat, loc, nbr, theta, theta_b):
        nbr32 = torch.as_tensor(nbr).to(feat.device, torch.int32)
        csr = _ops.csr_build(nbr32, 1, feat.shape[0])
        df, dth, dtb, dl = _ops.conv_backward(g, feat, loc, nbr32, csr, theta, theta_b, 1, feat.shape[0])
        return df, dth, dtb, dl

    return fwd, bwd


def sharded_forward(plan: HaloPlan, feat_local, loc_local, theta, theta_b, compute=None):
    """Owned rows of flex_conv on the local [owned | halo] buffers."""
    fwd, _ = compute or cuda_compute()
    return fwd(feat_local, loc_local, plan.local_nbr, theta, theta_b)[: plan.n_own]


def sharded_backward_local(plan: HaloPlan, g_owned, feat_local, loc_local, theta, theta_b, compute=None):
    """Local backward with zero upstream on the halo rows: returns the LOCAL partials
    (d_features [n_local, C], d_theta, d_theta_b, d_locations [n_local, d]); finish with
    scatter_halo_add on d_features / d_locations and fixed_order_allreduce on theta."""
    _, bwd = compute or cuda_compute()
    pad = torch.zeros((len(plan.halo),) + tuple(g_owned.shape[1:]), dtype=g_owned.dtype, device=g_owned.device)
    g_local = torch.cat([g_owned, pad], 0)
    return bwd(g_local, feat_local, loc_local, plan.local_nbr, theta, theta_b)

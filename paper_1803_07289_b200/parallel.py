"""Multi-GPU sharding of the flex-convolution hot path.

The reference is single-process (its only parallelism is OpenMP over points and a Python
loop over clouds with gradient accumulation, harness.py:589-599).  Two partitionings:

* Batch sharding (configs C2 / C5): clouds are independent units; rank r takes a
  contiguous block of clouds (`shard_range`).  The only collective is the theta / theta_b
  gradient sum of the training step, done by `fixed_order_allreduce`: all-gather, then sum
  in rank order in fp64 -- bitwise reproducible for a given world size (no float
  reduction-order nondeterminism).

* Point-chunk sharding of ONE large cloud with neighbour halos (configs C3 / C4, the
  north_star's 7M-point cloud over 8 GPUs): `ShardedCloud`.  Each rank holds a contiguous
  block of the spatially ordered cloud and never the global neighbour table:
    1. exact kNN of its own points with a POSITION GHOST SHELL -- a local kNN among the
       owned points bounds every point's k-th-neighbour distance by R (the rank's largest),
       so all true neighbours lie in the owned bounding box grown by R; each rank sends
       the others its points inside their grown boxes, and the kNN over [owned | ghosts]
       (ordered by global index, so index tie-breaking is the global one) gives the exact
       rows of the owned points (tests/test_parallel.py: equal to the unsharded table);
    2. the halo (neighbours owned elsewhere, a subset of the ghosts), the local neighbour
       table over [owned | halo], the reverse CSR and the exchange index lists, all device
       tensors built once per neighbourhood;
  then per layer: forward = halo gather of feature rows (one grouped point-to-point
  exchange, posted first; the interior rows -- all neighbours owned -- are computed while it
  is in flight, fc_conv_forward_rows, then the boundary rows) + the flex-conv kernels on the
  local buffers; backward = the local backward
  with zero upstream on the halo rows, the halo rows' d_features / d_locations partials
  sent back and added at the owners in fixed source-rank order, d_theta / d_theta_b summed
  by `fixed_order_allreduce` -- the only collective, and only for training.

Transport: torch.distributed grouped isend/irecv (NCCL over NVLink on the GPU box; gloo in
the CPU tests and for several ranks sharing one GPU, through host staging).
"""

from __future__ import annotations

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


# ---------------------------------------------------------------------------- transport
class Comm:
    """Grouped point-to-point exchange and all-gather over torch.distributed.  NCCL moves
    device tensors directly (NVLink); gloo (the CPU tests, or several ranks sharing one GPU)
    stages device tensors through host memory.  Zero-sized messages are skipped on both
    sides (their sizes are always agreed first)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        single = not (dist.is_available() and dist.is_initialized())
        self.rank = 0 if single else dist.get_rank(group)
        self.world = 1 if single else dist.get_world_size(group)
        self.host = (not single) and dist.get_backend(group) == "gloo"
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else \
                torch.device("cpu")
        self.wire = torch.device("cpu") if self.host else torch.device(device)

    def all_gather(self, t: torch.Tensor) -> list[torch.Tensor]:
        """Same-shape tensors from every rank, in rank order."""
        if self.world == 1:
            return [t]
        w = t.contiguous().to(self.wire)
        parts = [torch.empty_like(w) for _ in range(self.world)]
        self.dist.all_gather(parts, w, group=self.group)
        return [p.to(t.device) for p in parts]

    def ordered_sum(self, t: torch.Tensor) -> torch.Tensor:
        """Sum over ranks accumulated in rank order in fp64 (deterministic), in t's dtype."""
        if self.world == 1:
            return t
        acc = torch.zeros(t.shape, dtype=torch.float64, device=t.device)
        for p in self.all_gather(t):
            acc += p.to(torch.float64)
        return acc.to(t.dtype)

    def exchange(self, sends: dict, recv_shapes: dict, dtype, device) -> dict:
        """sends[r]: tensor for rank r; recv_shapes[r]: shape expected from rank r.
        Returns {r: received tensor on `device`} (empty tensors for zero-sized shapes)."""
        return self.exchange_finish(self.exchange_start(sends, recv_shapes, dtype, device))

    def exchange_start(self, sends: dict, recv_shapes: dict, dtype, device):
        """Post the grouped sends / receives and return at once (NCCL: the transfers run on
        the process group's stream while the caller keeps launching kernels); gloo completes
        here.  exchange_finish(handle) waits (stream-ordered for NCCL) and returns the rows."""
        ops, bufs, keep = [], {}, []
        for r, shape in recv_shapes.items():
            bufs[r] = torch.empty(shape, dtype=dtype, device=self.wire)
            if bufs[r].numel():
                ops.append(self.dist.P2POp(self.dist.irecv, bufs[r], r, self.group))
        for r, t in sends.items():
            if t.numel():
                w = t.contiguous().to(self.wire)
                keep.append(w)
                ops.append(self.dist.P2POp(self.dist.isend, w, r, self.group))
        reqs = self.dist.batch_isend_irecv(ops) if ops else []
        if self.host:  # gloo: blocking transport
            for req in reqs:
                req.wait()
            reqs = []
        return reqs, bufs, keep, device

    def exchange_finish(self, handle) -> dict:
        reqs, bufs, _keep, device = handle
        for req in reqs:
            req.wait()
        return {r: b.to(device) for r, b in bufs.items()}

    def exchange_sizes(self, counts: dict) -> dict:
        """counts[r] = number of items this rank will send to r; returns {r: number of items
        r will send here} for every other rank."""
        mine = torch.tensor([int(counts.get(r, 0)) for r in range(self.world)], dtype=torch.int64)
        table = self.all_gather(mine.to(self.wire))  # [world] rows of counts: table[src][dst]
        return {r: int(table[r][self.rank].item()) for r in range(self.world) if r != self.rank}


# ---------------------------------------------------------------------------- sharded cloud
def default_kernels():
    """The product kernels (libflexconv_b200.so): kNN, conv forward / backward, CSR."""
    from . import _ops

    def knn(points, k):
        return _ops.knn(points.contiguous(), 1, points.shape[0], k)

    def conv_fwd(feat, loc, nbr, theta, theta_b):
        return _ops.conv_forward(feat, loc, nbr, theta, theta_b, 1, feat.shape[0])

    def conv_bwd(g, feat, loc, nbr, csr, theta, theta_b, need):
        return _ops.conv_backward(g, feat, loc, nbr, csr, theta, theta_b, 1, feat.shape[0], need=need)

    def csr(nbr):
        return _ops.csr_build(nbr, 1, nbr.shape[0], validate=False)

    def conv_fwd_rows(feat, loc, nbr, theta, theta_b, rows, out):
        """None when the shape has no row-list kernel (the caller then runs the plain path)."""
        c_out, c_in, d = theta.shape
        if not _ops.conv_forward_rows_supported(c_in, d, nbr.shape[1], c_out, feat.dtype):
            return None
        return _ops.conv_forward_rows(feat, loc, nbr, theta, theta_b, rows, out)

    return {"knn": knn, "conv_fwd": conv_fwd, "conv_bwd": conv_bwd, "csr": csr, "conv_fwd_rows": conv_fwd_rows}


class ShardedCloud:
    """This rank's part of a point-chunk sharded cloud: owned rows [lo, hi) of the globally
    (spatially) ordered cloud plus the halo, with everything the layers need on the device.

    Local point ids: owned global g -> g - lo; halo[q] -> n_own + q.  `table` is the int32
    [n_own + n_halo, k] neighbour table over local ids (halo rows are self-loops: they carry
    zero upstream gradient and their forward outputs are discarded); `csr` its reverse.
    """

    def __init__(self):
        raise TypeError("use ShardedCloud.build(...)")

    @classmethod
    def build(cls, positions: torch.Tensor, k: int, comm: Comm, kernels=None) -> "ShardedCloud":
        """positions: this rank's owned points [n_own, d] (a contiguous block, in rank order,
        of the spatially ordered cloud).  Collective over `comm`."""
        self = object.__new__(cls)
        kern = kernels or default_kernels()
        self.comm, self.k, self.kernels = comm, int(k), kern
        rank, world = comm.rank, comm.world
        dev = positions.device
        pos = positions.contiguous()
        n_own, d = pos.shape
        sizes = [int(t.item()) for t in comm.all_gather(torch.tensor([n_own], dtype=torch.int64, device=dev))]
        self.bounds = [0]
        for s in sizes:
            self.bounds.append(self.bounds[-1] + s)
        self.lo, self.hi = self.bounds[rank], self.bounds[rank + 1]
        self.n_own, self.n_global = n_own, self.bounds[-1]
        if min(sizes) < self.k:
            raise ConfigInvalidError(f"every rank needs at least k={self.k} points (sizes {sizes})")

        # 1) ghost shell: R = the largest k-th-neighbour distance among owned points when only
        #    owned points are candidates (an upper bound on every owned point's true one).
        #    A rank's region is described by its occupied cells of a coarse global grid (a
        #    block of a Morton-type order is not a box); a point is a ghost for rank q when its
        #    cell lies within floor(R_q / cell) + 1 cells of one of q's occupied cells -- every
        #    true neighbour of q's points does (per-axis gap <= R_q).
        own_tab = kern["knn"](pos, self.k).long()
        p64 = pos.double()
        r2 = ((p64 - p64[own_tab[:, -1]]) ** 2).sum(dim=1).max()
        radius = torch.sqrt(r2) * (1.0 + 1e-9)
        metas = comm.all_gather(torch.cat([p64.min(dim=0).values, p64.max(dim=0).values, radius.reshape(1)]))
        gmin = torch.stack([m[:d] for m in metas]).min(dim=0).values
        gmax = torch.stack([m[d:2 * d] for m in metas]).max(dim=0).values
        cells_per_axis = int(min(64, max(4, round((self.n_global / 8) ** (1.0 / d)))))
        cs = torch.clamp((gmax - gmin) / cells_per_axis, min=1e-300)
        shape = (cells_per_axis,) * d + (1,) * (3 - d)

        def cell_ids(p):
            c = torch.clamp(((p - gmin) / cs).floor().long(), 0, cells_per_axis - 1)
            ids = c[:, 0]
            for t in range(1, d):
                ids = ids * cells_per_axis + c[:, t]
            return ids

        my_cells = cell_ids(p64)
        occ = torch.zeros(cells_per_axis ** d, dtype=torch.uint8, device=dev)
        occ[my_cells] = 1
        occs = comm.all_gather(occ)
        sends_pos, sends_gid = {}, {}
        for q in range(world):
            if q == rank:
                continue
            reach = int(torch.max(torch.floor(metas[q][2 * d] / cs)).item()) + 1
            grown = torch.nn.functional.max_pool3d(occs[q].view(1, 1, *shape).float(), kernel_size=tuple(
                2 * reach + 1 if s_ > 1 else 1 for s_ in shape), stride=1,
                padding=tuple(reach if s_ > 1 else 0 for s_ in shape)).flatten() > 0
            ids = torch.nonzero(grown[my_cells]).flatten()
            sends_pos[q] = pos[ids]
            sends_gid[q] = ids + self.lo
        counts = comm.exchange_sizes({q: t.shape[0] for q, t in sends_pos.items()})
        got_pos = comm.exchange(sends_pos, {q: (c, d) for q, c in counts.items()}, pos.dtype, dev)
        got_gid = comm.exchange(sends_gid, {q: (c,) for q, c in counts.items()}, torch.int64, dev)
        # candidates ordered by global id: ghosts of lower ranks, owned block, higher ranks
        before = [q for q in range(rank) if q in got_pos]
        after = [q for q in range(rank + 1, world) if q in got_pos]
        cand_pos = torch.cat([got_pos[q] for q in before] + [pos] + [got_pos[q] for q in after])
        own_gid = torch.arange(self.lo, self.hi, device=dev, dtype=torch.int64)
        cand_gid = torch.cat([got_gid[q] for q in before] + [own_gid] + [got_gid[q] for q in after])
        off = sum(got_pos[q].shape[0] for q in before)
        self.n_ghost = int(cand_pos.shape[0] - n_own)

        # 2) exact rows of the owned points, in global ids
        cand_tab = kern["knn"](cand_pos, self.k).long()
        rows = cand_gid[cand_tab[off:off + n_own]]
        self.global_rows = rows  # [n_own, k] global ids (inspection / tests)
        outside = (rows < self.lo) | (rows >= self.hi)
        self.halo = torch.unique(rows[outside])  # sorted global ids
        n_halo = int(self.halo.numel())
        self.n_local = n_own + n_halo
        local = torch.where(outside, n_own + torch.searchsorted(self.halo, rows), rows - self.lo)
        self_rows = (n_own + torch.arange(n_halo, device=dev, dtype=torch.int64))[:, None].expand(n_halo, self.k)
        self.table = torch.cat([local, self_rows]).to(torch.int32).contiguous()
        # halo positions come with the ghosts (no further exchange)
        self.positions = torch.cat([pos, cand_pos[torch.searchsorted(cand_gid, self.halo)]]).contiguous()

        # 3) exchange lists: the halo ids owned by rank q form a contiguous slice of `halo`
        bnd = torch.tensor(self.bounds, device=dev, dtype=torch.int64)
        cuts = torch.searchsorted(self.halo, bnd).tolist()
        self.recv_slices = {q: (cuts[q], cuts[q + 1]) for q in range(world) if q != rank and cuts[q + 1] > cuts[q]}
        req = {q: self.halo[a:b] - self.bounds[q] for q, (a, b) in self.recv_slices.items()}
        counts = comm.exchange_sizes({q: t.numel() for q, t in req.items()})
        got = comm.exchange(req, {q: (c,) for q, c in counts.items() if c > 0}, torch.int64, dev)
        self.send_idx = {q: t for q, t in got.items()}  # owned local ids rank q needs from here
        self.csr = kern["csr"](self.table)
        # interior rows (every neighbour owned) can be computed before the halo arrives
        bnd_mask = (self.table[:n_own] >= n_own).any(dim=1)
        self.interior_rows = torch.nonzero(~bnd_mask).flatten().to(torch.int32)
        self.boundary_rows = torch.nonzero(bnd_mask).flatten().to(torch.int32)
        return self

    # ------------------------------------------------------------------ row exchanges
    def local_buffer(self, owned: torch.Tensor) -> torch.Tensor:
        """A [n_local, C] buffer holding `owned` in its first n_own rows (halo rows zero).
        Layers exchange halo rows in place in such buffers, so a producer that writes its
        output straight into one (or a caller that keeps one) pays no per-call copy."""
        buf = torch.zeros((self.n_local,) + tuple(owned.shape[1:]), dtype=owned.dtype, device=owned.device)
        buf[: self.n_own] = owned
        return buf

    def fill_halo(self, local: torch.Tensor) -> torch.Tensor:
        """Fill the halo rows of a [n_local, C] buffer from their owners (in place)."""
        return self.fill_halo_finish(self.fill_halo_start(local))

    def fill_halo_start(self, local: torch.Tensor):
        """Post the halo exchange of `local` (returns at once with NCCL)."""
        c = tuple(local.shape[1:])
        h = self.comm.exchange_start({q: local[i] for q, i in self.send_idx.items()},
                                     {q: (b - a,) + c for q, (a, b) in self.recv_slices.items()}, local.dtype,
                                     local.device)
        return h, local

    def fill_halo_finish(self, handle) -> torch.Tensor:
        h, local = handle
        got = self.comm.exchange_finish(h)
        for q, (a, b) in self.recv_slices.items():
            local[self.n_own + a:self.n_own + b] = got[q]
        return local

    def gather(self, owned: torch.Tensor) -> torch.Tensor:
        """[n_own, C] owned rows -> a new [n_local, C] buffer with the halo rows filled."""
        return self.fill_halo(self.local_buffer(owned))

    def reduce_halo(self, local: torch.Tensor) -> torch.Tensor:
        """Add the other ranks' halo-row partials for this rank's points into the owned rows
        of `local` (in place; ascending source-rank order, indices unique per source:
        deterministic).  Returns the owned rows (a view)."""
        c = tuple(local.shape[1:])
        got = self.comm.exchange({q: local[self.n_own + a:self.n_own + b] for q, (a, b) in self.recv_slices.items()},
                                 {q: (i.numel(),) + c for q, i in self.send_idx.items()}, local.dtype, local.device)
        owned = local[: self.n_own]
        for q in sorted(got):
            owned.index_add_(0, self.send_idx[q], got[q])
        return owned

    def scatter_add(self, local: torch.Tensor) -> torch.Tensor:
        """reduce_halo on a copy (leaves `local` untouched)."""
        return self.reduce_halo(local.clone())

    @property
    def halo_fraction(self) -> float:
        return (self.n_local - self.n_own) / max(self.n_own, 1)


class ShardedFlexConv:
    """flex_conv on a ShardedCloud: owned rows of the forward, and the training backward
    (d_features / d_locations of the owned rows, d_theta / d_theta_b summed over ranks).

    Inputs may be owned rows ([n_own, C], copied into a local buffer per call) or local
    buffers ([n_local, C] from cloud.local_buffer: the features' halo rows are refreshed in
    place, the upstream gradient's halo rows must be zero) -- the latter is the copy-free
    path a multi-layer network uses."""

    def __init__(self, cloud: ShardedCloud):
        self.cloud = cloud
        self._saved = None

    def _local(self, t):
        return t if t.shape[0] == self.cloud.n_local else self.cloud.local_buffer(t)

    def forward(self, feat, theta, theta_b):
        """Owned rows of the forward.  With a row-list kernel (kernels["conv_fwd_rows"]) the
        interior rows -- whose neighbours are all owned -- are computed while the halo rows
        are in flight (posted before, waited for after), then the boundary rows."""
        cl = self.cloud
        pos = cl.positions if cl.positions.dtype == feat.dtype else cl.positions.to(feat.dtype)
        feat = self._local(feat)
        rows_k = cl.kernels.get("conv_fwd_rows")
        out = None
        if rows_k is not None:
            handle = cl.fill_halo_start(feat)
            buf = torch.empty((cl.n_local, theta.shape[0]), dtype=feat.dtype, device=feat.device)
            if rows_k(feat, pos, cl.table, theta, theta_b, cl.interior_rows, buf) is not None:
                cl.fill_halo_finish(handle)
                rows_k(feat, pos, cl.table, theta, theta_b, cl.boundary_rows, buf)
                out = buf
            else:
                cl.fill_halo_finish(handle)
        else:
            cl.fill_halo(feat)
        if out is None:
            out = cl.kernels["conv_fwd"](feat, pos, cl.table, theta, theta_b)
        self._saved = (feat, pos, theta, theta_b)
        return out[: cl.n_own]

    def backward(self, g, with_locations=True):
        cl = self.cloud
        feat, pos, theta, theta_b = self._saved
        self._saved = None
        df, dth, dtb, dl = cl.kernels["conv_bwd"](self._local(g), feat, pos, cl.table, cl.csr, theta, theta_b,
                                                  (True, True, True, bool(with_locations)))
        df = cl.reduce_halo(df)
        dl = cl.reduce_halo(dl) if with_locations else None
        grads = cl.comm.ordered_sum(torch.cat([dth.reshape(-1), dtb.reshape(-1)]))
        return df, grads[: dth.numel()].view_as(dth), grads[dth.numel():].view_as(dtb), dl

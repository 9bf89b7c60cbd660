"""Neighbourhood index and the exact kNN builder -- the reference's neighborhood API
(/root/reference/pkg/src/flexconv/neighborhood.py) on the B200 kNN kernels.

Row i of every neighbour table is [i, the k-1 nearest OTHER points by (squared distance,
index)] (neighborhood.py:1-8).  The reference answers queries from a CPU kd-tree; here
`build_kdtree` returns a lightweight spatial index over the point set and `knn_query`
runs the GPU grid/brute kNN (csrc/knn.cu), which produces bit-identical rows.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, _ops
from .errors import (
    ConfigInvalidError,
    EmptyInputError,
    IndexOutOfRangeError,
    NonFiniteError,
    ShapeMismatchError,
)

DEFAULT_LEAF_SIZE = 16


def _device():
    return torch.device("cuda", torch.cuda.current_device())


class NeighborIndex:
    """n x k table of neighbour indices; row i is [i, nearest others...]
    (neighborhood.py:54-71).  `indices` keeps the caller's type (numpy int64 as in the
    reference, or a torch tensor).  The device copy (int32, range-checked once) and the
    reverse neighbourhood are cached per device so repeated layers reuse them."""

    def __init__(self, indices):
        if isinstance(indices, torch.Tensor):
            if indices.dtype not in (torch.int32, torch.int64):
                indices = indices.to(torch.int64)
            self.indices = indices.contiguous()
        else:
            self.indices = np.ascontiguousarray(indices, dtype=np.int64)
        if self.indices.ndim != 2:
            raise ShapeMismatchError(f"indices must be 2-d, got shape {tuple(self.indices.shape)}")
        self._dev: dict = {}

    @property
    def n(self) -> int:
        return int(self.indices.shape[0])

    @property
    def k(self) -> int:
        return int(self.indices.shape[1])

    def device_table(self, device=None, n_points: int | None = None) -> torch.Tensor:
        """int32 [n, k] CUDA table; validates indices against [0, n_points) once
        (the reference's idx.min()/max() scan, flexops.py:92-93)."""
        device = device or _device()
        hi = self.n if n_points is None else int(n_points)
        key = (str(device), hi)
        hit = self._dev.get(key)
        if hit is not None:
            return hit["table"]
        src = self.indices
        if isinstance(src, np.ndarray):
            src = torch.from_numpy(src)
        src = src.to(device, non_blocking=False)
        if src.dtype == torch.int64:
            table, bad = _ops.narrow_indices(src, hi)
        else:
            table = src.contiguous()
            bad = _ops.check_indices(table, hi)
        if table.numel() and int(bad.item()) != 0:
            raise IndexOutOfRangeError("neighbor index out of [0, n)")
        self._dev[key] = {"table": table}
        return table

    def reverse(self, device=None, n_points: int | None = None):
        """Reverse neighbourhood (CSR) on `device`, built once."""
        device = device or _device()
        hi = self.n if n_points is None else int(n_points)
        table = self.device_table(device, hi)
        entry = self._dev[(str(device), hi)]
        if "csr" not in entry:  # the table was range-checked by device_table: no host sync here
            entry["csr"] = _ops.csr_build(table, 1, hi, validate=False)
        return entry["csr"]


def _check_locations(locations):
    """Coerce/validate a location matrix (neighborhood.py:75-83)."""
    if isinstance(locations, torch.Tensor):
        if locations.dim() != 2:
            raise ShapeMismatchError(f"locations must be n x d, got shape {tuple(locations.shape)}")
        if locations.shape[0] == 0:
            raise EmptyInputError("no points to index")
        if not bool(torch.isfinite(locations).all()):
            raise NonFiniteError("locations contain NaN or Inf")
        return locations
    locations = np.ascontiguousarray(locations, dtype=np.float64)
    if locations.ndim != 2:
        raise ShapeMismatchError(f"locations must be n x d, got shape {locations.shape}")
    if locations.shape[0] == 0:
        raise EmptyInputError("no points to index")
    if not np.isfinite(locations).all():
        raise NonFiniteError("locations contain NaN or Inf")
    return locations


@dataclass
class KdTree:
    """Spatial index handle returned by `build_kdtree` (the reference's KdTree,
    neighborhood.py:29-51, is a CPU structure; the GPU kNN bins points into a uniform
    grid per query call, so the handle only carries the point set it was built on)."""

    points: object
    leaf_size: int = DEFAULT_LEAF_SIZE
    depth: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.points.shape[0])


def build_kdtree(locations, leaf_size: int = DEFAULT_LEAF_SIZE) -> KdTree:
    """Drop-in for neighborhood.build_kdtree (neighborhood.py:85-146)."""
    points = _check_locations(locations)
    if leaf_size < 1:
        raise ConfigInvalidError(f"leaf_size must be >= 1, got {leaf_size}")
    points = points.clone() if isinstance(points, torch.Tensor) else points.copy()
    return KdTree(points=points, leaf_size=leaf_size)


def _run_knn(locations, k: int, algo: int) -> NeighborIndex:
    is_np = not isinstance(locations, torch.Tensor)
    pts = torch.from_numpy(locations) if is_np else locations
    dev = pts.device if pts.is_cuda else _device()
    pts = pts.to(dev)
    if pts.dtype not in (torch.float32, torch.float64):
        pts = pts.to(torch.float64)
    n = pts.shape[0]
    if not 1 <= k <= n:
        raise ConfigInvalidError(f"k must satisfy 1 <= k <= {n}, got {k}")
    out = _ops.knn(pts, 1, n, int(k), algo)
    if is_np:
        return NeighborIndex(out.to(torch.int64).cpu().numpy())
    nb = NeighborIndex(out.to(torch.int64) if not locations.is_cuda else out)
    nb._dev[(str(dev), n)] = {"table": out}
    return nb


def knn_query(tree: KdTree, locations, k: int, num_threads: int = 1) -> NeighborIndex:
    """Exact kNN rows for the index's own points (neighborhood.py:149-168).
    `num_threads` is accepted for signature compatibility and ignored."""
    locations = _check_locations(locations)
    same = (locations.shape == tree.points.shape)
    if same:
        if isinstance(locations, torch.Tensor) or isinstance(tree.points, torch.Tensor):
            a = torch.as_tensor(locations)
            b = torch.as_tensor(tree.points).to(a.device)
            same = bool(torch.equal(a, b.to(a.dtype)))
        else:
            same = np.array_equal(locations, tree.points)
    if not same:
        raise ShapeMismatchError("locations differ from the points the tree was built on")
    return _run_knn(locations, k, _lib.KNN_AUTO)


def knn_brute_force(locations, k: int) -> NeighborIndex:
    """O(n^2) scan with the same contract as knn_query (neighborhood.py:171-187)."""
    locations = _check_locations(locations)
    return _run_knn(locations, k, _lib.KNN_BRUTE)


def validate_neighbors(locations, neighbors: NeighborIndex) -> None:
    """Check all NeighborIndex invariants against its point set (neighborhood.py:190-208).
    Host-side checker (test utility, as in the reference)."""
    locations = np.asarray(torch.as_tensor(_check_locations(locations)).cpu(), dtype=np.float64)
    idx = np.asarray(torch.as_tensor(neighbors.indices).cpu(), dtype=np.int64)
    n = locations.shape[0]
    if idx.shape[0] != n:
        raise ShapeMismatchError(f"index has {idx.shape[0]} rows for {n} points")
    if idx.min() < 0 or idx.max() >= n:
        raise IndexOutOfRangeError("neighbor index out of [0, n)")
    if not (idx[:, 0] == np.arange(n)).all():
        raise IndexOutOfRangeError("row i must start with i itself")
    for i in range(n):
        row = idx[i]
        if len(np.unique(row)) != len(row):
            raise IndexOutOfRangeError(f"row {i} has duplicate entries")
        d2 = ((locations[i] - locations[row[1:]]) ** 2).sum(axis=-1)
        keys = list(zip(d2.tolist(), row[1:].tolist()))
        if keys != sorted(keys):
            raise IndexOutOfRangeError(f"row {i} not sorted by (distance, index)")


# the reference keeps its file formats in these modules; same names here
from .formats import read_neighbors, write_neighbors  # noqa: E402,F401  (neighborhood.py:211-252)

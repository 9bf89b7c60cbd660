"""Inverse-density importance subsampling (IDISS) and resolution hierarchies -- the
reference's sampling API (/root/reference/pkg/src/flexconv/sampling.py) on the GPU.

* `inverse_density` runs `fc_inverse_density` (csrc/knn.cu): fp64 in the reference's numpy
  evaluation order, bitwise equal to sampling.py:33-48.
* `idiss_sample` draws the exponential race keys from the caller's `Rng` on the host (the
  reference's Philox stream, so the draws are identical), divides by phi on the device and
  keeps the m smallest keys with a stable device sort (ties -> lower index, the order of
  `np.lexsort((arange, keys))`, sampling.py:51-72).
* `build_hierarchy` chains GPU kNN levels (`knn_query`, bit-identical rows) exactly as
  sampling.py:112-146 does.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _ops
from .core import PointCloud, Rng, validate_cloud
from .errors import ConfigInvalidError, IndexOutOfRangeError, ShapeMismatchError
from .neighborhood import DEFAULT_LEAF_SIZE, NeighborIndex, build_kdtree, knn_query


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def inverse_density(locations, neighbors: NeighborIndex):
    """phi[i] = sum of Euclidean distances from point i to its neighbour row (the self
    entry contributes zero), sampling.py:33-48.  numpy in -> numpy out; a CUDA tensor in ->
    a CUDA fp64 tensor out."""
    is_np = not isinstance(locations, torch.Tensor)
    loc = torch.from_numpy(np.ascontiguousarray(locations, dtype=np.float64)) if is_np else locations
    n = int(loc.shape[0])
    if neighbors.n != n:
        raise ShapeMismatchError(f"neighbor index has {neighbors.n} rows for {n} points")
    dev = loc.device if loc.is_cuda else _device()
    loc = loc.to(device=dev, dtype=torch.float64).contiguous()
    phi = _ops.inverse_density(loc, neighbors.device_table(dev, n))
    return phi.cpu().numpy() if is_np else phi


def idiss_sample(phi, m: int, rng: Rng) -> np.ndarray:
    """Draw m distinct indices with first-draw probability phi[i] / sum(phi) by exponential
    race keys (key_i = Exp(1) / phi_i, keep the m smallest), sampling.py:51-72.  Returns the
    sorted selection as int64 numpy (the reference's type)."""
    is_np = not isinstance(phi, torch.Tensor)
    phi_t = torch.from_numpy(np.asarray(phi, dtype=np.float64)) if is_np else phi.to(torch.float64)
    n = int(phi_t.shape[0])
    if not 1 <= m <= n:
        raise ConfigInvalidError(f"m must satisfy 1 <= m <= {n}, got {m}")
    dev = phi_t.device if phi_t.is_cuda else _device()
    phi_t = phi_t.to(dev)
    if bool((phi_t < 0).any()):
        raise ConfigInvalidError("phi must be nonnegative")
    if not bool((phi_t != 0).any()):
        warnings.warn("all-zero density: falling back to uniform sampling", RuntimeWarning)
        return random_sample(n, m, rng)
    draws = torch.from_numpy(rng.gen.exponential(size=n)).to(dev)
    keys = draws / phi_t  # IEEE division: x / 0 = inf, as numpy under errstate(divide="ignore")
    order = torch.sort(keys, stable=True).indices[:m]
    return torch.sort(order).values.to(torch.int64).cpu().numpy()


def random_sample(n: int, m: int, rng: Rng) -> np.ndarray:
    """Uniform without-replacement baseline (sampling.py:75-79): the draw is the caller's
    host RNG stream, as in the reference."""
    if not 1 <= m <= n:
        raise ConfigInvalidError(f"m must satisfy 1 <= m <= {n}, got {m}")
    return np.sort(rng.gen.choice(n, size=m, replace=False)).astype(np.int64)


@dataclass
class HierarchyLevel:
    """One resolution: its cloud, its own neighbourhoods and (except at level 0) the
    selected indices into the parent level (sampling.py:82-89)."""

    cloud: PointCloud
    neighbors: NeighborIndex
    selection: np.ndarray | None
    parent_n: int | None = None  # size of the level the selection indexes
    _dev: dict = field(default_factory=dict, repr=False)

    def device(self, dtype=torch.float64, device=None) -> dict:
        """Device copies used by the network layers (built once per dtype/device):
        locations [n, d], the int32 neighbour table and the int32 selection."""
        device = device or _device()
        key = (str(device), dtype)
        hit = self._dev.get(key)
        if hit is None:
            hit = {"locations": torch.from_numpy(self.cloud.locations).to(device=device, dtype=dtype).contiguous(),
                   "table": self.neighbors.device_table(device, self.cloud.n)}
            if self.selection is not None:
                hit["selection"] = torch.from_numpy(np.asarray(self.selection, dtype=np.int64)).to(device)
                sel32, bad = _ops.narrow_indices(hit["selection"], self.parent_n if self.parent_n is not None else 2 ** 31 - 1)
                if hit["selection"].numel() and int(bad.item()):
                    raise IndexOutOfRangeError("selection index out of [0, n_parent)")
                hit["selection32"] = sel32
            self._dev[key] = hit
        return hit


@dataclass
class ResolutionHierarchy:
    levels: list[HierarchyLevel]
    k: int
    factor: int
    mode: str

    @property
    def depth(self) -> int:
        return len(self.levels) - 1

    def sizes(self) -> list[int]:
        return [lv.cloud.n for lv in self.levels]


def spatially_ordered(cloud: PointCloud, *per_point):
    """Data preparation: the cloud's points (and any per-point arrays, e.g. labels) permuted
    into cell order (ops.spatial_order).  Flex-convolution is permutation equivariant
    (reference tests/test_flexops.py:263-276), and idiss_sample returns sorted indices, so
    every level of a hierarchy built from the reordered cloud is spatially ordered too: the
    neighbour rows of consecutive points then share cache lines (the gathers hit L1/L2)
    instead of landing anywhere in the cloud.  Returns (cloud, *per_point, perm)."""
    pos = torch.from_numpy(np.ascontiguousarray(cloud.locations)).to(_device(), torch.float64)
    perm = _ops.spatial_order(pos).to(torch.int64).cpu().numpy()
    out = [PointCloud(cloud.locations[perm], cloud.features[perm])]
    out += [np.asarray(a)[perm] for a in per_point]
    return (*out, perm)


def concat_hierarchies(hierarchies: list[ResolutionHierarchy]) -> ResolutionHierarchy:
    """Several scenes' hierarchies as ONE hierarchy of disjoint clouds: level t holds the
    scenes' level-t points back to back, neighbour rows and selections shifted by each
    scene's offset.  No neighbourhood crosses a scene, so every operator of the network
    computes exactly the per-scene results; one launch then covers all scenes (used by
    network.train_step_batch(fused=True) for a GPU's share of the batch)."""
    if not hierarchies:
        raise ConfigInvalidError("no hierarchies to concatenate")
    h0 = hierarchies[0]
    depth = h0.depth
    if any(h.depth != depth or h.k != h0.k for h in hierarchies):
        raise ShapeMismatchError("hierarchies must share depth and k")
    levels = []
    for t in range(depth + 1):
        locs, feats, nbrs, sels = [], [], [], []
        off = par_off = 0
        for h in hierarchies:
            lv = h.levels[t]
            locs.append(lv.cloud.locations)
            feats.append(lv.cloud.features)
            idx = lv.neighbors.indices
            idx = idx.cpu().numpy() if isinstance(idx, torch.Tensor) else np.asarray(idx)
            nbrs.append(idx.astype(np.int64) + off)
            if t:
                sels.append(np.asarray(lv.selection, dtype=np.int64) + par_off)
                par_off += h.levels[t - 1].cloud.n
            off += lv.cloud.n
        cloud = PointCloud(np.concatenate(locs), np.concatenate(feats))
        selection = np.concatenate(sels) if t else None
        levels.append(HierarchyLevel(cloud, NeighborIndex(np.concatenate(nbrs)), selection,
                                     par_off if t else None))
    return ResolutionHierarchy(levels, k=h0.k, factor=h0.factor, mode=h0.mode)


def _level_neighbors(locations, k: int, num_threads: int, leaf_size: int) -> NeighborIndex:
    tree = build_kdtree(locations, leaf_size)
    return knn_query(tree, tree.points, min(k, locations.shape[0]), num_threads)


def build_hierarchy(cloud: PointCloud, k: int, factor: int, depth: int, rng: Rng,
                    mode: str = "idiss", num_threads: int = 1,
                    leaf_size: int = DEFAULT_LEAF_SIZE) -> ResolutionHierarchy:
    """Chain of subsampled levels; level t keeps ceil(n / factor^t) points, each with a
    fresh neighbourhood over its own points (sampling.py:112-146)."""
    validate_cloud(cloud)
    if factor < 2:
        raise ConfigInvalidError(f"factor must be >= 2, got {factor}")
    if depth < 1:
        raise ConfigInvalidError(f"depth must be >= 1, got {depth}")
    if mode not in ("idiss", "random"):
        raise ConfigInvalidError(f"mode must be 'idiss' or 'random', got {mode!r}")
    if cloud.n < factor ** depth:
        raise ConfigInvalidError(f"n={cloud.n} too small for factor={factor}, depth={depth}")
    levels = [HierarchyLevel(cloud, _level_neighbors(cloud.locations, k, num_threads, leaf_size), None)]
    for t in range(1, depth + 1):
        parent = levels[-1]
        m = -(-cloud.n // factor ** t)  # ceil division
        level_rng = rng.spawn(t)
        if mode == "idiss":
            phi = inverse_density(parent.device()["locations"], parent.neighbors)
            selection = idiss_sample(phi, m, level_rng)
        else:
            selection = random_sample(parent.cloud.n, m, level_rng)
        sub = PointCloud(parent.cloud.locations[selection], parent.cloud.features[selection])
        levels.append(HierarchyLevel(sub, _level_neighbors(sub.locations, k, num_threads, leaf_size), selection,
                                     parent.cloud.n))
    return ResolutionHierarchy(levels, k=k, factor=factor, mode=mode)


# the reference keeps its file formats in these modules; same names here
from .formats import load_hierarchy, save_hierarchy  # noqa: E402,F401  (sampling.py:149-204)

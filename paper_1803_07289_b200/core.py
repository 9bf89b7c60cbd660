"""Core containers and the deterministic RNG used for synthetic inputs.

`Rng` restates the reference's Philox generator with derivable substreams
(/root/reference/pkg/src/flexconv/core.py:86-112) so the benchmark and the tests draw
exactly the inputs the reference harness would draw for the same seed.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import EmptyInputError, NonFiniteError, ShapeMismatchError

_MIX = 0x9E3779B97F4A7C15  # splitmix64 increment (core.py:86)


@dataclass
class Rng:
    """Counter-based Philox RNG; `spawn(tag)` derives an independent stream (core.py:89-107)."""

    seed: int
    stream: int = 0
    gen: np.random.Generator = field(init=False, repr=False)

    def __post_init__(self):
        key = [int(self.seed) % 2 ** 64, int(self.stream) % 2 ** 64]
        self.gen = np.random.Generator(np.random.Philox(key=key))

    def spawn(self, tag: int) -> "Rng":
        return Rng(self.seed, (self.stream * _MIX + int(tag) + 1) % 2 ** 64)


def _as_matrix(a, name: str) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ShapeMismatchError(f"{name} must be 2-d, got shape {a.shape}")
    return a


@dataclass
class PointCloud:
    """n points: locations (n, d) plus features (n, C), coerced to float64 (core.py:29-55)."""

    locations: np.ndarray
    features: np.ndarray

    def __post_init__(self):
        self.locations = _as_matrix(self.locations, "locations")
        self.features = _as_matrix(self.features, "features")

    @property
    def n(self) -> int:
        return self.locations.shape[0]

    @property
    def d(self) -> int:
        return self.locations.shape[1]

    @property
    def C(self) -> int:
        return self.features.shape[1]


def validate_cloud(cloud: PointCloud) -> None:
    """Raise unless all PointCloud invariants hold (core.py:115-129)."""
    loc, feat = cloud.locations, cloud.features
    if loc.shape[0] != feat.shape[0]:
        raise ShapeMismatchError(f"locations have {loc.shape[0]} rows but features have {feat.shape[0]}")
    if loc.shape[0] < 1:
        raise EmptyInputError("point cloud has no points")
    if loc.shape[1] < 1 or feat.shape[1] < 1:
        raise ShapeMismatchError("d and C must both be >= 1")
    if not np.isfinite(loc).all():
        raise NonFiniteError("locations contain NaN or Inf")
    if not np.isfinite(feat).all():
        raise NonFiniteError("features contain NaN or Inf")


def lattice_positions(gen: np.random.Generator, n: int, d: int) -> np.ndarray:
    """Uniform U[0,1)^d positions snapped to the 2^-24 grid: exactly
    representable in fp32, and every fp64 squared distance between two of them is exact,
    so kNN ties are real ties and fp32/fp64 runs see identical inputs."""
    return np.floor(gen.uniform(0.0, 1.0, size=(n, d)) * 2.0 ** 24) / 2.0 ** 24


def synthetic_layer(seed: int, tag: int, n: int, d: int, c_in: int, c_out: int):
    """Synthetic flex-conv layer inputs of SURVEY.md §8(d): positions on the 2^-24 lattice,
    features / upstream N(0,1) and theta / theta_b 0.1*N(0,1), all cast to fp32 values
    (returned as float64 arrays holding fp32-representable numbers)."""
    g = Rng(seed).spawn(tag).gen
    loc = lattice_positions(g, n, d)
    feat = g.standard_normal((n, c_in)).astype(np.float32).astype(np.float64)
    theta = (g.standard_normal((c_out, c_in, d)) * 0.1).astype(np.float32).astype(np.float64)
    theta_b = (g.standard_normal((c_out, c_in)) * 0.1).astype(np.float32).astype(np.float64)
    up = g.standard_normal((n, c_out)).astype(np.float32).astype(np.float64)
    return loc, feat, theta, theta_b, up


# the reference keeps its file formats in these modules; same names here
from .formats import read_cloud, write_cloud  # noqa: E402,F401  (core.py:148-219)

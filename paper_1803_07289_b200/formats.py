"""The reference's on-disk formats, byte-compatible in both directions:

* flexcloud  (/root/reference/pkg/src/flexconv/core.py:148-219): ASCII header
  "flexcloud v1 n d C" / "flexcloud-labeled v1 n d C", then one line per point with the d
  locations and C features as shortest round-trip reals (Python repr), plus an int label.
* flexknn    (neighborhood.py:211-252): "flexknn v1 n k" + n lines of k integers.
* flexhier   (sampling.py:149-204): a directory with level<t>.cloud / level<t>.knn per level
  and a sorted-key, indent-1 JSON manifest holding k, factor, mode and the selections.

Same headers, separators, number formatting and validation order as the reference, so files
written here are byte-identical to the reference's and either side reads the other's; the
same EngineError subclasses are raised for the same defects.  Parsing is vectorised over the
whole body (one split per line, one numpy conversion) instead of a per-value Python loop.
(flexckpt, the checkpoint format, lives with the network: network.save/load_checkpoint.)
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .core import PointCloud, validate_cloud
from .errors import (
    ConfigInvalidError,
    EmptyInputError,
    IndexOutOfRangeError,
    IoFailureError,
    NonFiniteError,
    ShapeMismatchError,
)


def _read_lines(path, what):
    try:
        with open(path) as fh:
            return fh.read().splitlines()
    except OSError as exc:
        raise IoFailureError(f"cannot read {what} file {path}: {exc}") from exc


def _fields(path, lines, want):
    """Split every body line; the first line with the wrong field count is reported with the
    reference's message (1-based file line numbers, header = line 1)."""
    rows = [ln.split() for ln in lines]
    for i, parts in enumerate(rows):
        if len(parts) != want:
            raise ConfigInvalidError(f"{path}: line {i + 2} has {len(parts)} fields, expected {want}")
    return rows


def _first_bad(path, rows, convs):
    """Raise the reference's per-line error for the first line with a malformed value;
    convs(parts) converts one line's fields (raising ValueError)."""
    for i, parts in enumerate(rows):
        try:
            convs(parts)
        except ValueError as exc:
            raise ConfigInvalidError(f"{path}: line {i + 2} has a malformed value") from exc
    raise ConfigInvalidError(f"{path}: malformed value")


# ------------------------------------------------------------------ flexcloud
def write_cloud(path, cloud: PointCloud, labels=None) -> None:
    """core.py:161-179."""
    validate_cloud(cloud)
    if labels is not None:
        labels = np.asarray(labels)
        if labels.shape != (cloud.n,):
            raise ShapeMismatchError(f"labels must have shape ({cloud.n},), got {labels.shape}")
        labels = labels.astype(np.int64)
    name = "flexcloud-labeled" if labels is not None else "flexcloud"
    vals = np.concatenate([cloud.locations, cloud.features], axis=1).tolist()
    out = [f"{name} v1 {cloud.n} {cloud.d} {cloud.C}\n"]
    if labels is None:
        out += [" ".join(map(repr, row)) + "\n" for row in vals]
    else:
        out += [" ".join(map(repr, row)) + " " + str(int(lab)) + "\n" for row, lab in zip(vals, labels.tolist())]
    try:
        with open(path, "w", newline="\n") as fh:
            fh.write("".join(out))
    except OSError as exc:
        raise IoFailureError(f"cannot write cloud file {path}: {exc}") from exc


def read_cloud(path):
    """core.py:182-219.  Returns (PointCloud, labels-or-None)."""
    lines = _read_lines(path, "cloud")
    if not lines:
        raise ConfigInvalidError(f"{path}: empty file")
    head = lines[0].split()
    if len(head) != 5 or head[0] not in ("flexcloud", "flexcloud-labeled") or head[1] != "v1":
        raise ConfigInvalidError(f"{path}: malformed header {lines[0]!r}")
    labeled = head[0] == "flexcloud-labeled"
    try:
        n, d, c = (int(t) for t in head[2:5])
    except ValueError as exc:
        raise ConfigInvalidError(f"{path}: non-integer sizes in header") from exc
    if n < 1 or d < 1 or c < 1:
        raise EmptyInputError(f"{path}: header declares n={n} d={d} C={c}")
    if len(lines) - 1 != n:
        raise ConfigInvalidError(f"{path}: header declares {n} points, file has {len(lines) - 1}")
    rows = _fields(path, lines[1:], d + c + (1 if labeled else 0))
    try:
        data = np.array([[float(t) for t in r[: d + c]] for r in rows], dtype=np.float64).reshape(n, d + c)
        labels = np.array([int(r[d + c]) for r in rows], dtype=np.int64) if labeled else None
    except ValueError:
        _first_bad(path, rows, lambda r: ([float(t) for t in r[: d + c]], [int(t) for t in r[d + c:]]))
    if not np.isfinite(data).all():
        raise NonFiniteError(f"{path}: non-finite value in data")
    return PointCloud(data[:, :d], data[:, d:]), labels


# ------------------------------------------------------------------ flexknn
def write_neighbors(path, neighbors) -> None:
    """neighborhood.py:214-221."""
    idx = neighbors.indices
    idx = idx.cpu().numpy() if hasattr(idx, "cpu") else np.asarray(idx)
    n, k = idx.shape
    body = [" ".join(map(str, row)) + "\n" for row in idx.astype(np.int64).tolist()]
    try:
        with open(path, "w", newline="\n") as fh:
            fh.write(f"flexknn v1 {n} {k}\n" + "".join(body))
    except OSError as exc:
        raise IoFailureError(f"cannot write neighbor file {path}: {exc}") from exc


def read_neighbors(path):
    """neighborhood.py:224-252."""
    from .neighborhood import NeighborIndex

    lines = _read_lines(path, "neighbor")
    if not lines:
        raise ConfigInvalidError(f"{path}: empty file")
    head = lines[0].split()
    if len(head) != 4 or head[0] != "flexknn" or head[1] != "v1":
        raise ConfigInvalidError(f"{path}: malformed header {lines[0]!r}")
    try:
        n, k = int(head[2]), int(head[3])
    except ValueError as exc:
        raise ConfigInvalidError(f"{path}: non-integer sizes in header") from exc
    if n < 1 or k < 1 or len(lines) - 1 != n:
        raise ConfigInvalidError(f"{path}: header sizes do not match file body")
    rows = _fields(path, lines[1:], k)
    try:
        idx = np.array([[int(t) for t in r] for r in rows], dtype=np.int64).reshape(n, k)
    except ValueError:
        _first_bad(path, rows, lambda r: [int(t) for t in r])
    if idx.min() < 0 or idx.max() >= n:
        raise IndexOutOfRangeError(f"{path}: neighbor index out of range")
    return NeighborIndex(idx)


# ------------------------------------------------------------------ flexhier
def save_hierarchy(hierarchy, out_dir) -> None:
    """sampling.py:152-179."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    manifest = {"format": "flexhier", "version": 1, "k": hierarchy.k, "factor": hierarchy.factor,
                "mode": hierarchy.mode, "levels": []}
    for t, lv in enumerate(hierarchy.levels):
        cloud_file, knn_file = f"level{t}.cloud", f"level{t}.knn"
        write_cloud(out / cloud_file, lv.cloud)
        write_neighbors(out / knn_file, lv.neighbors)
        manifest["levels"].append({"n": lv.cloud.n, "cloud": cloud_file, "knn": knn_file,
                                   "selection": None if lv.selection is None else
                                   [int(v) for v in np.asarray(lv.selection).tolist()]})
    try:
        with open(out / "manifest.json", "w", newline="\n") as fh:
            json.dump(manifest, fh, sort_keys=True, indent=1)
            fh.write("\n")
    except OSError as exc:
        raise IoFailureError(f"cannot write manifest: {exc}") from exc


def load_hierarchy(in_dir):
    """sampling.py:182-204."""
    from .sampling import HierarchyLevel, ResolutionHierarchy

    path = Path(in_dir) / "manifest.json"
    try:
        with open(path) as fh:
            manifest = json.load(fh)
    except OSError as exc:
        raise IoFailureError(f"cannot read manifest {path}: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise ConfigInvalidError(f"{path}: invalid JSON: {exc}") from exc
    if manifest.get("format") != "flexhier" or manifest.get("version") != 1:
        raise ConfigInvalidError(f"{path}: not a flexhier v1 manifest")
    levels = []
    for t, entry in enumerate(manifest["levels"]):
        cloud, _ = read_cloud(Path(in_dir) / entry["cloud"])
        neighbors = read_neighbors(Path(in_dir) / entry["knn"])
        sel = entry["selection"]
        selection = None if sel is None else np.asarray(sel, dtype=np.int64)
        if (t == 0) != (selection is None):
            raise ConfigInvalidError(f"{path}: level {t} selection map inconsistent")
        parent_n = None if t == 0 else levels[-1].cloud.n
        levels.append(HierarchyLevel(cloud, neighbors, selection, parent_n))
    return ResolutionHierarchy(levels, k=int(manifest["k"]), factor=int(manifest["factor"]),
                               mode=str(manifest["mode"]))

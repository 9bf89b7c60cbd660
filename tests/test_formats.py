"""The reference's file formats (flexcloud, flexknn, flexhier) against files the REFERENCE
wrote (tests/golden/formats/, made by tests/golden/make_format_golden.py): byte-identical
output, identical parse, the reference's exception classes for malformed files
(reference tests: /root/reference/pkg/tests/test_core.py, test_neighborhood.py)."""

import filecmp
import os

import numpy as np
import pytest

from conftest import GOLDEN

FMT = os.path.join(GOLDEN, "formats")


@pytest.fixture(scope="module")
def arrays():
    with np.load(os.path.join(FMT, "arrays.npz")) as z:
        return {k: z[k] for k in z.files}


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


def test_cloud_byte_identical_and_round_trip(tmp_path, arrays):
    from paper_1803_07289_b200 import core

    cloud = core.PointCloud(arrays["loc"], arrays["feats"])
    core.write_cloud(tmp_path / "a.cloud", cloud)
    assert _bytes(tmp_path / "a.cloud") == _bytes(os.path.join(FMT, "cloud.cloud"))
    core.write_cloud(tmp_path / "b.cloud", cloud, arrays["labels"])
    assert _bytes(tmp_path / "b.cloud") == _bytes(os.path.join(FMT, "labeled.cloud"))
    got, lab = core.read_cloud(os.path.join(FMT, "labeled.cloud"))
    np.testing.assert_array_equal(got.locations, arrays["loc"])  # shortest repr round-trips exactly
    np.testing.assert_array_equal(got.features, arrays["feats"])
    np.testing.assert_array_equal(lab, arrays["labels"])
    got, lab = core.read_cloud(os.path.join(FMT, "cloud.cloud"))
    assert lab is None and got.n == arrays["loc"].shape[0]


def test_neighbors_byte_identical_and_round_trip(tmp_path, arrays):
    from paper_1803_07289_b200 import neighborhood

    nb = neighborhood.read_neighbors(os.path.join(FMT, "cloud.knn"))
    np.testing.assert_array_equal(np.asarray(nb.indices), arrays["nbr"])
    neighborhood.write_neighbors(tmp_path / "a.knn", nb)
    assert _bytes(tmp_path / "a.knn") == _bytes(os.path.join(FMT, "cloud.knn"))
    neighborhood.write_neighbors(tmp_path / "b.knn", neighborhood.NeighborIndex(arrays["nbr"]))
    assert _bytes(tmp_path / "b.knn") == _bytes(os.path.join(FMT, "cloud.knn"))


def test_hierarchy_load_save_byte_identical(tmp_path):
    from paper_1803_07289_b200 import sampling

    h = sampling.load_hierarchy(os.path.join(FMT, "hier"))
    assert h.sizes() == [500, 125, 32] and (h.k, h.factor, h.mode) == (8, 4, "idiss")
    assert h.levels[1].parent_n == 500 and h.levels[2].parent_n == 125
    sampling.save_hierarchy(h, tmp_path / "h")
    names = sorted(os.listdir(os.path.join(FMT, "hier")))
    assert sorted(os.listdir(tmp_path / "h")) == names
    _, mismatch, errors = filecmp.cmpfiles(os.path.join(FMT, "hier"), tmp_path / "h", names, shallow=False)
    assert not mismatch and not errors


@pytest.mark.parametrize("body, exc", [
    ("", "ConfigInvalidError"),
    ("flexcloud v2 1 1 1\n0 0\n", "ConfigInvalidError"),
    ("flexcloud v1 x 1 1\n0 0\n", "ConfigInvalidError"),
    ("flexcloud v1 0 1 1\n", "EmptyInputError"),
    ("flexcloud v1 2 1 1\n0 0\n", "ConfigInvalidError"),
    ("flexcloud v1 2 1 1\n0 0\n1\n", "ConfigInvalidError"),
    ("flexcloud v1 2 1 1\n0 0\n1 zz\n", "ConfigInvalidError"),
    ("flexcloud v1 2 1 1\n0 0\n1 inf\n", "NonFiniteError"),
    ("flexcloud-labeled v1 1 1 1\n0 0 1.5\n", "ConfigInvalidError"),
])
def test_cloud_errors(tmp_path, body, exc):
    from paper_1803_07289_b200 import core, errors

    p = tmp_path / "bad.cloud"
    p.write_text(body)
    with pytest.raises(getattr(errors, exc)):
        core.read_cloud(p)


@pytest.mark.parametrize("body, exc", [
    ("", "ConfigInvalidError"),
    ("flexknn v1 2 2\n0 1\n", "ConfigInvalidError"),
    ("flexknn v1 2 2\n0 1\n1\n", "ConfigInvalidError"),
    ("flexknn v1 2 2\n0 1\n1 q\n", "ConfigInvalidError"),
    ("flexknn v1 2 2\n0 1\n1 2\n", "IndexOutOfRangeError"),
])
def test_neighbor_errors(tmp_path, body, exc):
    from paper_1803_07289_b200 import errors, neighborhood

    p = tmp_path / "bad.knn"
    p.write_text(body)
    with pytest.raises(getattr(errors, exc)):
        neighborhood.read_neighbors(p)


def test_missing_files_raise_io_failure(tmp_path):
    from paper_1803_07289_b200 import core, errors, neighborhood, sampling

    for fn in (core.read_cloud, neighborhood.read_neighbors, sampling.load_hierarchy):
        with pytest.raises(errors.IoFailureError):
            fn(tmp_path / "nope")

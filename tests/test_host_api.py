"""Host-side pieces of the reference API that need no GPU: param_count
(flexops.py:64-67), FlexConvParams validation (flexops.py:22-51) and validate_neighbors
(neighborhood.py:190-208) on the reference's own kNN rows (tests/golden/knn.npz)."""

import numpy as np
import pytest

from conftest import load_golden


def test_param_count():
    from paper_1803_07289_b200 import param_count

    assert param_count(64, 64, 3) == 16384  # C'·C·(d+1)
    assert param_count(32, 32, 3) == 4096
    assert param_count(3, 2, 1) == 12


def test_flex_conv_params_validation():
    from paper_1803_07289_b200 import FlexConvParams
    from paper_1803_07289_b200.errors import NonFiniteError, ShapeMismatchError

    p = FlexConvParams(np.zeros((4, 3, 2)), np.zeros((4, 3)))
    assert (p.c_out, p.c_in, p.d) == (4, 3, 2)
    with pytest.raises(ShapeMismatchError):
        FlexConvParams(np.zeros((4, 3, 2)), np.zeros((3, 4)))
    with pytest.raises(ShapeMismatchError):
        FlexConvParams(np.zeros((4, 3)), np.zeros((4, 3)))
    with pytest.raises(NonFiniteError):
        FlexConvParams(np.full((1, 1, 1), np.inf), np.zeros((1, 1)))


@pytest.mark.parametrize("case", ["ties_n300_d2_k7", "uniform_n57_d1_k5", "uniform_n1000_d3_k8", "dups_n4_d2_k4"])
def test_validate_neighbors_accepts_reference_rows(case):
    from paper_1803_07289_b200 import NeighborIndex, validate_neighbors

    g = load_golden("knn.npz")
    validate_neighbors(g[f"{case}__points"], NeighborIndex(g[f"{case}__indices"]))


def test_validate_neighbors_rejects_corrupt_rows():
    from paper_1803_07289_b200 import NeighborIndex, validate_neighbors
    from paper_1803_07289_b200.errors import IndexOutOfRangeError, ShapeMismatchError

    g = load_golden("knn.npz")
    pts, idx = g["uniform_n200_d2_k9__points"], g["uniform_n200_d2_k9__indices"]
    bad = idx.copy()
    bad[5, 0] = 6  # row does not start with itself
    with pytest.raises(IndexOutOfRangeError):
        validate_neighbors(pts, NeighborIndex(bad))
    bad = idx.copy()
    bad[5, 2] = bad[5, 1]  # duplicate entry
    with pytest.raises(IndexOutOfRangeError):
        validate_neighbors(pts, NeighborIndex(bad))
    bad = idx.copy()
    bad[5, 1], bad[5, 2] = idx[5, 2], idx[5, 1]  # not sorted by (distance, index)
    with pytest.raises(IndexOutOfRangeError):
        validate_neighbors(pts, NeighborIndex(bad))
    bad = idx.copy()
    bad[7, 3] = 200  # out of range
    with pytest.raises(IndexOutOfRangeError):
        validate_neighbors(pts, NeighborIndex(bad))
    with pytest.raises(ShapeMismatchError):
        validate_neighbors(pts[:-1], NeighborIndex(idx))

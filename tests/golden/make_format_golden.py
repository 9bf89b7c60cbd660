"""Golden files of the reference's on-disk formats, written by the REFERENCE itself
(core.write_cloud, neighborhood.write_neighbors, sampling.save_hierarchy) into
tests/golden/formats/.  Run here (where /root/reference exists):
    python tests/golden/make_format_golden.py
tests/test_formats.py checks that paper_1803_07289_b200.formats writes byte-identical files
and reads them back to identical arrays."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402

OUT = os.path.join(HERE, "formats")


def main():
    fc = import_reference()
    from flexconv import core, neighborhood, sampling

    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(3)
    n = 300
    loc = rng.random((n, 3)) * np.array([1.0, 1e-7, 3e5])
    loc[:5] = [[0.1, 0.2, 0.3], [1e-300, 5e-324, -0.0], [1.5e20, -2.0, 7.0], [1 / 3, 2 / 3, 1.0], [0.0, 1e16, 123456789.123]]
    feats = rng.standard_normal((n, 2))
    cloud = core.PointCloud(loc, feats)
    core.write_cloud(os.path.join(OUT, "cloud.cloud"), cloud)
    labels = rng.integers(0, 7, n)
    core.write_cloud(os.path.join(OUT, "labeled.cloud"), cloud, labels)
    nbr = neighborhood.knn_brute_force(loc, 6)
    neighborhood.write_neighbors(os.path.join(OUT, "cloud.knn"), nbr)
    h = sampling.build_hierarchy(core.PointCloud(rng.random((500, 3)), rng.standard_normal((500, 1))), 8, 4, 2,
                                 core.Rng(5).spawn(1))
    sampling.save_hierarchy(h, os.path.join(OUT, "hier"))
    np.savez(os.path.join(OUT, "arrays.npz"), loc=loc, feats=feats, labels=labels, nbr=np.asarray(nbr.indices))
    print("wrote", sorted(os.listdir(OUT)), fc.__name__)


if __name__ == "__main__":
    main()

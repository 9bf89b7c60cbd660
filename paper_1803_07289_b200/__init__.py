"""paper_1803_07289_b200 -- B200-native (sm_100a) Flex-Convolution hot path.

Drop-in for the reference package's operator surface (flexconv.flexops /
flexconv.neighborhood, /root/reference/pkg/src/flexconv/__init__.py:20-37) plus the
north_star batched torch ops (flex_conv / flex_pool / flex_deconv / knn on [B, D, N]).
All arithmetic runs in libflexconv_b200.so (hand-written CUDA for sm_100a); importing
the package without the built library raises (there is no CPU fallback).
"""

from . import _lib

_lib.lib()  # fail loudly at import if the CUDA library is missing

from . import backend  # noqa: E402
from .core import PointCloud, Rng, validate_cloud  # noqa: E402
from .errors import (  # noqa: E402
    ConfigInvalidError,
    EmptyInputError,
    EngineError,
    IndexOutOfRangeError,
    IoFailureError,
    NonFiniteError,
    ShapeMismatchError,
)
from .flexops import (  # noqa: E402
    FlexConvParams,
    GradBundle,
    downsample_gather,
    flex_conv_backward,
    flex_conv_forward,
    flex_deconv_forward,
    flex_max_pool,
    flex_max_pool_backward,
    flex_upsample,
    param_count,
    pointwise_conv,
    pointwise_conv_backward,
    scatter_to_fine,
)
from .neighborhood import (  # noqa: E402
    KdTree,
    NeighborIndex,
    build_kdtree,
    knn_brute_force,
    knn_query,
    validate_neighbors,
)
from .ops import Neighborhood, flex_conv, flex_deconv, flex_pool, knn, spatial_order  # noqa: E402

__version__ = "0.1.0"

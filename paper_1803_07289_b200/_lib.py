"""ctypes binding of the C ABI (include/flexconv_b200.h) -> libflexconv_b200.so.

This is the only way the package reaches the GPU: there is no CPU fallback and no
second backend.  If the shared library is missing the import fails loudly.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
# FC_LIB_PATH: A/B timing of an alternative build (scripts/*_probe.py); defaults to the in-tree library
LIB_PATH = os.environ.get("FC_LIB_PATH") or os.path.join(HERE, "libflexconv_b200.so")

FC_F32, FC_F64 = 0, 1
MODE_AUTO, MODE_SIMT, MODE_TC_SPLIT, MODE_TC_BF16 = 0, 1, 2, 3
KNN_AUTO, KNN_BRUTE, KNN_GRID = 0, 1, 2

_STATUS = {
    1: errors.ShapeMismatchError,
    2: errors.IndexOutOfRangeError,
    3: errors.NonFiniteError,
    4: errors.EmptyInputError,
    5: errors.ConfigInvalidError,
    6: errors.CudaError,
    7: errors.UnsupportedError,
}

# name -> argtypes (restype is int unless listed in _RESTYPE)
_P, _I64, _I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
SIGNATURES = {
    "fc_abi_version": [],
    "fc_last_error": [],
    "fc_launch_count": [],
    "fc_profile_enable": [_I],
    "fc_profile_reset": [],
    "fc_profile_count": [],
    "fc_profile_name": [_I],
    "fc_profile_ms": [_I],
    "fc_conv_forward": [_I, _I, _I64, _I64, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P],
    "fc_conv_backward": [_I, _I, _I64, _I64, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "fc_conv_forward_rows": [_I64, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _I64, _P, _P],
    "fc_deconv_backward": [_I, _I, _I64, _I64, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "fc_scratch_peak_bytes": [],
    "fc_scratch_peak_reset": [],
    "fc_deconv_forward": [_I, _I, _I64, _I64, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "fc_csr_build": [_I64, _I64, _I, _P, _P, _P, _P],
    "fc_csr_build_async": [_I64, _I64, _I, _P, _P, _P, _P, _P],
    "fc_pool_forward": [_I, _I64, _I64, _I, _I, _P, _P, _P, _P, _P],
    "fc_pool_backward": [_I, _I64, _I64, _I, _I, _P, _P, _P, _P, _P, _P],
    "fc_record_csr_build": [_I64, _I64, _I, _P, _P, _P, _P],
    "fc_pool_backward_record": [_I, _I64, _I64, _I, _P, _P, _P, _P, _P],
    "fc_knn": [_I, _I64, _I64, _I, _I, _P, _P, _I, _P],
    "fc_spatial_order": [_I, _I64, _I, _P, _P, _P],
    "fc_inverse_density": [_I64, _I, _I, _P, _P, _P, _P],
    "fc_gather_rows": [_I, _I64, _I, _P, _P, _P, _P],
    "fc_scatter_rows": [_I, _I64, _I64, _I, _P, _P, _P, _P],
    "fc_selection_owner": [_I64, _I64, _P, _P, _P],
    "fc_pool_select_forward": [_I, _I64, _I64, _I, _I, _P, _P, _P, _P, _P, _P, _P],
    "fc_pool_select_backward": [_I, _I64, _I64, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "fc_indices_to_i32": [_P, _P, _I64, _I64, _P, _P],
    "fc_check_indices": [_P, _I64, _I64, _P, _P],
    "fc_count_nonfinite": [_I, _P, _I64, _P, _P],
    "fc_gemm_image_bytes": [_I, _I],
    "fc_gemm_pack_b": [_I, _I, _I, _P, _P, _P, _I64, _P, _P],
    "fc_gemm_rows": [_I64, _I, _P, _P, _P, _P, _I64, _P, _I, _P, _I, _P, _P, _P, _P, _P, _I64, _P],
    "fc_gemm_wgrad": [_I64, _P, _I64, _P, _I64, _I, _I, _P, _P, _P, _P, _P, _P],
    "fc_relu_backward": [_I, _I64, _P, _P, _P, _P, _P],
}
_RESTYPE = {"fc_last_error": ctypes.c_char_p, "fc_launch_count": ctypes.c_uint64, "fc_profile_enable": None,
            "fc_profile_reset": None, "fc_profile_name": ctypes.c_char_p, "fc_profile_ms": ctypes.c_float,
            "fc_gemm_image_bytes": ctypes.c_int64, "fc_scratch_peak_bytes": ctypes.c_int64,
            "fc_scratch_peak_reset": None}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1803_07289_b200.build` "
                "(there is no CPU fallback)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = handle
    return _lib


def call(name: str, *args) -> None:
    """Invoke an entry point; map a non-zero status to the reference's exception class."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().fc_last_error().decode(errors="replace")
        raise _STATUS.get(rc, errors.EngineError)(f"{name}: {msg}")


def launch_count() -> int:
    return int(lib().fc_launch_count())


class KernelTimer:
    """Context manager: per-kernel CUDA-event times recorded by the library on the
    launching stream (fc_profile_*).  `.times` maps kernel name -> list of ms."""

    def __enter__(self):
        lib().fc_profile_reset()
        lib().fc_profile_enable(1)
        self.times = {}
        return self

    def __exit__(self, *exc):
        import torch

        lib().fc_profile_enable(0)
        torch.cuda.synchronize()
        for i in range(lib().fc_profile_count()):
            name = lib().fc_profile_name(i).decode()
            self.times.setdefault(name, []).append(float(lib().fc_profile_ms(i)))
        lib().fc_profile_reset()


def symbols() -> list[str]:
    return list(SIGNATURES)

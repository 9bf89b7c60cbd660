"""CPU: the C-ABI library builds for sm_100a, loads without a GPU, and exports every
entry point include/flexconv_b200.h declares; the Python binding covers all of them and
maps status codes onto the reference's exception classes.  No compute calls."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "flexconv_b200.h")
LIB = os.path.join(ROOT, "paper_1803_07289_b200", "libflexconv_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|float|const char \*|uint64_t|int64_t)\s*(fc_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_1803_07289_b200 import build

        build.build(verbose=False)
    return ctypes.CDLL(LIB)


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for must in ("fc_conv_forward", "fc_conv_backward", "fc_deconv_forward", "fc_pool_forward",
                 "fc_pool_backward", "fc_knn", "fc_csr_build", "fc_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_python_binding_covers_header():
    from paper_1803_07289_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_abi_version_and_error_string(lib):
    lib.fc_abi_version.restype = ctypes.c_int
    assert lib.fc_abi_version() == 1
    lib.fc_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.fc_last_error(), bytes)


def test_validation_errors_without_gpu():
    """Argument validation happens before any device work, so it runs on a CPU host."""
    from paper_1803_07289_b200 import _lib, errors

    with pytest.raises(errors.EmptyInputError):
        _lib.call("fc_conv_forward", 0, 0, 1, 0, 4, 3, 8, 4, None, None, None, None, None, None, None)
    with pytest.raises(errors.ShapeMismatchError):
        _lib.call("fc_conv_forward", 0, 0, 1, 10, 0, 3, 8, 4, None, None, None, None, None, None, None)
    with pytest.raises(errors.ConfigInvalidError):
        _lib.call("fc_knn", 0, 1, 10, 3, 11, None, None, 0, None)
    with pytest.raises(errors.ConfigInvalidError):
        _lib.call("fc_conv_forward", 7, 0, 1, 10, 4, 3, 8, 4, None, None, None, None, None, None, None)


def test_sass_is_sm100a():
    """The shipped cubin targets sm_100a (checked with cuobjdump when available)."""
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe) or not os.path.exists(LIB):
        pytest.skip("cuobjdump or library missing")
    out = subprocess.run([exe, "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out

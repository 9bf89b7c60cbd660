#!/usr/bin/env bash
# Build the UNMODIFIED reference kernels (flexconv._native, Cython -> C -> gcc)
# straight from the read-only reference tree into oracle/_ref/.
#
# Test/bench infrastructure only: nothing under oracle/ is on the product path.
# Recipe mirrors /root/reference/pkg/setup.py:5-14 (-O3 -fopenmp, numpy include),
# but runs cython + gcc directly instead of the reference's setuptools build.
# Output: oracle/_ref/_native.<EXT_SUFFIX>, importable as top-level `_native`.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${FLEXCONV_REF:-/root/reference/pkg/src/flexconv}"
OUT="$HERE/_ref"
if [ ! -f "$REF/_native.pyx" ]; then
  echo "build_ref: reference source $REF/_native.pyx not present; skipping" >&2
  exit 0
fi
mkdir -p "$OUT"
PY=${PYTHON:-python}
SUFFIX=$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')
PYINC=$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')
NPINC=$($PY -c 'import numpy; print(numpy.get_include())')
# cython writes the generated C into oracle/_ref (git-ignored); the .pyx is read in place.
$PY -m cython -3 --module-name _native -o "$OUT/_native.c" "$REF/_native.pyx"
# /opt/gcc (the image default $CC) lacks libgomp.spec; the system gcc has OpenMP.
CC=${REF_CC:-/usr/bin/gcc}
$CC -O3 -fopenmp -fPIC -shared -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -I"$PYINC" -I"$NPINC" "$OUT/_native.c" -o "$OUT/_native$SUFFIX"
echo "build_ref: built $OUT/_native$SUFFIX"
# Pack the reference package and its own test suite next to the build output (git-ignored,
# travels to the GPU box like the .so; a tarball, so no reference source lies in the tree):
# tests/test_gpu_ref_suite.py unpacks it and runs the reference's test_flexops.py /
# test_neighborhood.py with the B200 module in the kernel slot.
PKG="$(dirname "$REF")"          # .../pkg/src
TESTS="$(dirname "$PKG")/tests"  # .../pkg/tests
STAGE="$(mktemp -d)"
mkdir -p "$STAGE/refpkg/flexconv" "$STAGE/refpkg/tests"
cp "$REF"/*.py "$STAGE/refpkg/flexconv/"
cp "$OUT/_native$SUFFIX" "$STAGE/refpkg/flexconv/_native$SUFFIX"
if [ -d "$TESTS" ]; then cp "$TESTS"/*.py "$STAGE/refpkg/tests/"; fi
tar -czf "$OUT/refsuite.tar.gz" -C "$STAGE" refpkg
rm -rf "$STAGE" "$OUT/refpkg"
echo "build_ref: packed the reference package + tests into $OUT/refsuite.tar.gz"

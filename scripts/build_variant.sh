#!/bin/bash
# A/B builds: compile the current csrc/ with some files replaced by other versions into a
# separate library (loaded with FC_LIB_PATH=... for side-by-side timing on one box).
#   bash scripts/build_variant.sh <out.so> [<csrc-file>=<path-or-git-rev:path> ...]
set -e
OUT=$(realpath -m "$1"); shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=$(mktemp -d)
mkdir -p $W/pkg $W/include
cp -r $ROOT/paper_1803_07289_b200/csrc $W/pkg/
cp $ROOT/include/*.h $W/include/
for spec in "$@"; do
  f=${spec%%=*}; src=${spec#*=}
  if [[ "$src" == *:* ]]; then git -C $ROOT show "$src" > $W/pkg/csrc/$f; else cp "$src" $W/pkg/csrc/$f; fi
done
cd $W/pkg/csrc
for f in *.cu; do
  /usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++ -c $f -o ${f%.cu}.o -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I $W/include -gencode arch=compute_100a,code=sm_100a ${NVCC_EXTRA:-} &
done
wait
/usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++ -shared -o $OUT *.o -gencode arch=compute_100a,code=sm_100a \
  -lcudart -lcuda -Xlinker -rpath=/usr/local/cuda/lib64
rm -rf $W
echo "built $OUT"

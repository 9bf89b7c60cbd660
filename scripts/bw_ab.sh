# usage: bash scripts/bw_ab.sh "name=lib ..." -- the 7M bandwidth kernels (bench_configs --only BW) per library build
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  if [ "$lib" = cur ]; then unset FC_LIB_PATH; else export FC_LIB_PATH=$PWD/$lib; fi
  timeout 300 python scripts/bench_configs.py --only BW 2>/dev/null | python -c "import json,sys
d=json.load(sys.stdin)['BW']; print('$name', {k: v['ms'] for k, v in d.items() if isinstance(v, dict)})"
done

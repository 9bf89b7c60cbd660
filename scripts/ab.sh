# usage: bash /tmp/ab.sh "name=lib ..."  (lib path relative to repo, or "cur")
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  if [ "$lib" = cur ]; then unset FC_LIB_PATH; else export FC_LIB_PATH=$PWD/$lib; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-fp64 > gpurun_out/ab_$name.log 2>&1
  tail -1 gpurun_out/ab_$name.log | python -c "import json,sys
try:
  l=json.loads(sys.stdin.read()); print('$name', l['ms_per_step'], {k:v['ms'] for k,v in l['roofline']['kernels'].items()})
except Exception as e: print('$name FAILED', e)"
done

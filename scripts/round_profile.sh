#!/bin/bash
# Round measurement bundle (GPU box): GPU tests, the bench line, the ncu launch list, one
# `ncu --set full` capture of the three headline kernels, and the per-kernel DRAM traffic.
#   bash scripts/round_profile.sh <tag>      (outputs under gpurun_out/, tag e.g. r01_v5)
set -u
TAG=${1:-run}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 $OUT/bench_$TAG.log > $OUT/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
# headline kernels (one launch each) + the grid-kNN query kernel (bench.py calls the kNN four
# times before the first step, so it is captured by its own -c 1 filter)
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:fwd64w|dt64|rev64w' -c 3 \
    -o $OUT/prof_$TAG -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:knn_grid_query' -c 1 \
    -o $OUT/prof_knn_$TAG -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-fp64 > /dev/null 2>&1; echo "ncu knn rc=$?"
timeout 600 python scripts/ncu_traffic.py > $OUT/ncu_traffic_$TAG.log 2>&1; echo "traffic rc=$?"
timeout 300 python scripts/ncu_datapipe.py $OUT/prof_$TAG.ncu-rep $OUT/prof_knn_$TAG.ncu-rep --out $OUT/ncu_datapipe_$TAG.json > /dev/null 2>&1; echo "datapipe rc=$?"
(timeout 300 python scripts/ncu_summary.py $OUT/prof_$TAG.ncu-rep; timeout 300 python scripts/ncu_summary.py $OUT/prof_knn_$TAG.ncu-rep) > $OUT/ncu_full_$TAG.txt 2>&1; echo "summary rc=$?"

#!/bin/bash
# Profiles judged for a round (run on the GPU box from the repo root):
#   1. plain bench (no profiler) -> gpurun_out/<R>_bench.json
#   2. ncu launch list of the same command (cold-cache, serialised)
#   3. ncu --set full of one timed config-2 k_raycast_pruned launch
# usage: tools/profile_round.sh r1
set -u
R=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
ARGS="--steps 3 --warmup 3 --no-extra --no-cpu-baseline"
python bench.py $ARGS > $OUT/${R}_bench.json 2> $OUT/${R}_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${R}_launches_bench.csv python bench.py $ARGS > $OUT/${R}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "bench_step/" \
    -k regex:k_raycast_pruned -s 3 -c 1 -o $OUT/${R}_k_raycast_pruned_full -f \
    python bench.py $ARGS > $OUT/${R}_ncu_full.log 2>&1
tail -2 $OUT/${R}_ncu_full.log

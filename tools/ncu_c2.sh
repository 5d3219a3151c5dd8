#!/bin/bash
# One ncu --set full capture (with source) of a timed config-2 k_raycast_pruned launch.
OUT=gpurun_out; mkdir -p $OUT
ARGS="--steps 3 --warmup 3 --no-extra --no-cpu-baseline"
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "bench_step/" \
    -k regex:k_raycast_pruned -s 3 -c 1 -o $OUT/${1:-c2}_pruned_full -f \
    python bench.py $ARGS > $OUT/${1:-c2}_ncu_full.log 2>&1
tail -2 $OUT/${1:-c2}_ncu_full.log

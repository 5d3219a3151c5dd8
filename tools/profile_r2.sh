#!/bin/bash
# Round-2 profiles (run on the GPU box from the repo root):
#   1. plain bench (no profiler)                  -> gpurun_out/r2_bench.json
#   2. ncu launch list of the config-2 bench      -> gpurun_out/r2_launches_bench.csv
#   3. ncu --set full of one timed k_raycast_pruned launch (config 2)
#   4. per-kernel metrics over configs 2/4/1/3/5  -> gpurun_out/r2_kernels.csv
set -u
OUT=gpurun_out
mkdir -p $OUT
ARGS="--steps 3 --warmup 3 --no-extra --no-cpu-baseline"
timeout 1500 python bench.py > $OUT/r2_bench.json 2> $OUT/r2_bench.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/r2_launches_bench.csv python bench.py $ARGS > $OUT/r2_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "bench_step/" \
    -k regex:k_raycast_pruned -s 3 -c 1 -o $OUT/r2_k_raycast_pruned_full -f \
    python bench.py $ARGS > $OUT/r2_ncu_full.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 2400 ncu --metrics $M --clock-control none --csv --print-units base -k regex:^k_ \
    --log-file $OUT/r2_kernels.csv python tools/kernel_table_run.py > $OUT/r2_kt.log 2>&1
tail -2 $OUT/r2_kt.log

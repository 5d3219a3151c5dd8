#!/bin/bash
# Build a debug copy of the library with VR_STATS event counters into $OUT
set -e
OUT=paper_2405_10050_b200/build/stats; mkdir -p $OUT
for f in paper_2405_10050_b200/csrc/*.cu; do
  nvcc -std=c++17 -O3 -DVR_STATS -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --cudart static -c $f -o $OUT/$(basename $f .cu).o &
done
wait
nvcc -shared --cudart static -gencode arch=compute_100a,code=sm_100a $OUT/*.o -o $OUT/_voronray_b200.so

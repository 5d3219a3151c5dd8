#!/bin/bash
# A/B of library variants: tools/ab_variant.sh name1 name2 ...
# name "base" = the in-tree library, otherwise paper_2405_10050_b200/_variant_<name>.so
# AB_WHICH = sweep_pruned.py workloads (default c2vert); AB_C5=1 adds the config-5 / config-4 runs.
for v in "$@"; do
  if [ $v = base ]; then unset VR_LIB_PATH; else export VR_LIB_PATH=$PWD/paper_2405_10050_b200/_variant_$v.so; fi
  echo "== $v"
  CHECK=1 MODES=pruned REPS=7 timeout 600 python tools/sweep_pruned.py ${AB_WHICH:-c2vert} 2>&1 | grep -v "^pool"
  if [ -n "$AB_C5" ]; then timeout 600 python tools/c5_ab.py 3 2>&1 | tail -2; fi
done

#!/bin/bash
# Round-2 final measurement: GPU tests, bench (ours), reference arm.
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/r2f_pytest.log 2>&1; echo "pytest rc $?" >> $OUT/r2f_pytest.log
timeout 1500 python bench.py > $OUT/r2f_bench.json 2> $OUT/r2f_bench.err; echo "bench rc $?" >> $OUT/r2f_bench.err
timeout 900 python bench.py --impl reference > $OUT/r2f_ref.json 2> $OUT/r2f_ref.err
tail -2 $OUT/r2f_pytest.log; tail -c 400 $OUT/r2f_bench.json; echo; cat $OUT/r2f_ref.json

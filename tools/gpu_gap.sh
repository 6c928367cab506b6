#!/bin/bash
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python tools/composite_gap.py 4 > $OUT/gap.log 2>&1; echo "gap exit $?" >> $OUT/status
timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "c5 exit $?" >> $OUT/status

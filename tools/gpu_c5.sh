#!/bin/bash
# C5 bench line + C5 sampled parity test + A/B of a variant on C4.
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
for v in ${2:-}; do
  RC_LIB=$PWD/paper_1809_01334_b200/librc_$v.so timeout 600 python bench.py --config 4 --steps 5 --no-cpu-baseline > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  echo "bench $v exit $?" >> $OUT/status
done
timeout 600 python bench.py --config 4 --steps 5 --no-cpu-baseline > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench default exit $?" >> $OUT/status
timeout 1200 python bench.py --config 5 --steps 2 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 exit $?" >> $OUT/status
timeout 1500 python -m pytest tests -m gpu -x -q -rA -k "c5 or fold" > $OUT/pytest_c5.log 2>&1; echo "pytest c5 exit $?" >> $OUT/status

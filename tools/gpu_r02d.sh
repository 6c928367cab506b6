#!/bin/bash
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
python tools/peaks.py $OUT/peaks.json > $OUT/peaks.log 2>&1; echo "peaks exit $?" >> $OUT/status
timeout 1800 python -m pytest tests -m gpu -q -rA -x -k "comm or debug_pair or bench_two or composite" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/status
timeout 900 python bench.py --steps 5 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench exit $?" >> $OUT/status

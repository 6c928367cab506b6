#!/bin/bash
# Parity subset, the composite probe and the default bench (no CPU baseline): bash tools/gpu_check.sh TAG "PYTEST_K"
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -k "$2" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/status
timeout 600 python tools/composite_gap.py 4 > $OUT/gap.log 2>&1; echo "gap exit $?" >> $OUT/status
for r in 1 2; do
  timeout 900 python bench.py --steps 5 --no-cpu-baseline > $OUT/bench_c4_$r.json 2> $OUT/bench_c4_$r.err; echo "bench $r exit $?" >> $OUT/status
done

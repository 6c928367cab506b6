#!/bin/bash
# Parity of the default build (skipped when PYTEST_K is "-"), then an interleaved A/B (two rounds)
# of librc variants on the bench: bash tools/gpu_ab2.sh TAG CONFIG PYTEST_K variant...
# variant "default" = librc.so, else paper_1809_01334_b200/librc_<variant>.so
set -u
TAG=$1; CFG=$2; K=$3; shift 3
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ "$K" != "-" ]; then
  timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_fold_gpu.py -m gpu -q -x -k "$K" > $OUT/pytest.log 2>&1
  echo "pytest exit $?" >> $OUT/status
fi
for r in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then LIB=""; else LIB=$PWD/paper_1809_01334_b200/librc_$v.so; fi
    RC_LIB=$LIB timeout 900 python bench.py --config $CFG --steps 5 --no-cpu-baseline --no-e2e > $OUT/bench_${v}_$r.json 2> $OUT/bench_${v}_$r.err
    echo "$v run $r exit $?" >> $OUT/status
  done
done

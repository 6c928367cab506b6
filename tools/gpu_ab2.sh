#!/bin/bash
# Parity of the default build, then an interleaved A/B (A B A B) of librc variants on the bench:
#   bash tools/gpu_ab2.sh TAG CONFIG PYTEST_K variant_a variant_b
set -u
TAG=$1; CFG=$2; K=$3; A=$4; B=$5
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_fold_gpu.py -m gpu -q -x -k "$K" > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/status
for r in 1 2; do
  for v in $A $B; do
    if [ "$v" = default ]; then LIB=""; else LIB=$PWD/paper_1809_01334_b200/librc_$v.so; fi
    RC_LIB=$LIB timeout 900 python bench.py --config $CFG --steps 5 --no-cpu-baseline --no-e2e > $OUT/bench_${v}_$r.json 2> $OUT/bench_${v}_$r.err
    echo "$v run $r exit $?" >> $OUT/status
  done
done

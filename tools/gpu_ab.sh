#!/bin/bash
# A/B of librc build variants on the bench (no CPU baseline): bash tools/gpu_ab.sh TAG CONFIG variant...
# variant "default" = librc.so, else paper_1809_01334_b200/librc_<variant>.so
set -u
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
for v in "$@"; do
  if [ "$v" = default ]; then LIB=""; else LIB=$PWD/paper_1809_01334_b200/librc_$v.so; fi
  RC_LIB=$LIB timeout 900 python bench.py --config $CFG --steps 5 --no-cpu-baseline > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  echo "$v exit $?" >> $OUT/status
done

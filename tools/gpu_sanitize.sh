#!/bin/bash
# compute-sanitizer evidence: one tool per call (B200_PROFILING.md).  bash tools/gpu_sanitize.sh TAG TOOL
set -u
OUT=gpurun_out/$1; TOOL=$2; mkdir -p $OUT
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 --error-exitcode 9 python tools/sanitize.py \
  > $OUT/sanitize_$TOOL.log 2>&1
echo "sanitize $TOOL exit $?" >> $OUT/status

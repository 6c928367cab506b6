#!/bin/bash
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
PCMD="python tools/profile_frame.py --config 55 --frames 1"
timeout 600 $PCMD > $OUT/plain_agg.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_coarsen_fast' -s 2 -c 1 \
    -o $OUT/agg $PCMD > $OUT/ncu_agg.log 2>&1
echo "ncu agg exit $?" >> $OUT/status

#!/bin/bash
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
PCMD="python tools/profile_frame.py --config 45 --frames 2"
timeout 300 $PCMD > $OUT/plain_pf.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_prep_slots' -s 1 -c 1 \
    -o $OUT/prep $PCMD > $OUT/ncu_prep.log 2>&1
echo "ncu prep exit $?" >> $OUT/status

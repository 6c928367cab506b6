#!/bin/bash
# C5 aggregation study: records / times per fold level, and ncu of the full-size aggregation kernels
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python tools/fold_levels_probe.py 5 5 > $OUT/fold_probe_c5.log 2>&1
echo "probe exit $?" >> $OUT/status
PCMD="python tools/profile_frame.py --config 5 --frames 1"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_coarsen_fast|k_scatter' -s 0 -c 2 \
    -o $OUT/agg_c5 $PCMD > $OUT/ncu_agg_c5.log 2>&1
echo "ncu agg c5 exit $?" >> $OUT/status

#!/bin/bash
# Peaks, one `ncu --set full` capture of the segment kernel at C4s (source-level), the DRAM
# traffic of the segment kernel at full C4, and the launch list of the default bench command.
# bash tools/gpu_prof.sh TAG [what: all|full|traffic|launches]
set -u
OUT=gpurun_out/$1; WHAT=${2:-all}; mkdir -p $OUT
python tools/peaks.py $OUT/peaks.json > $OUT/peaks.log 2>&1; echo "peaks exit $?" >> $OUT/status
if [ "$WHAT" = all ] || [ "$WHAT" = full ]; then
  PCMD="python tools/profile_frame.py --config 45 --frames 2"
  timeout 300 $PCMD > $OUT/plain_pf.log 2>&1 && \
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_cast_curved' -s 1 -c 1 \
      -o $OUT/prof $PCMD > $OUT/ncu_full.log 2>&1
  echo "ncu full exit $?" >> $OUT/status
fi
if [ "$WHAT" = all ] || [ "$WHAT" = traffic ]; then
  TCMD="python tools/profile_frame.py --config 4 --frames 3"
  timeout 600 $TCMD > $OUT/plain_traffic.log 2>&1 && \
    timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:'k_cast_curved' -s 2 -c 1 --csv --log-file $OUT/traffic_c4.csv $TCMD > $OUT/ncu_traffic.log 2>&1
  echo "traffic exit $?" >> $OUT/status
fi
if [ "$WHAT" = all ] || [ "$WHAT" = launches ]; then
  CMD="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 900 $CMD > $OUT/plain.log 2>&1 && \
    timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|rc::' --csv \
      --log-file $OUT/launches_c4.csv $CMD > $OUT/ncu_launches.log 2>&1
  echo "launches exit $?" >> $OUT/status
fi

#!/bin/bash
# launch list (per-kernel device times) of the bench command: bash tools/gpu_launch.sh TAG [CONFIG]
set -u
OUT=gpurun_out/$1; CFG=${2:-4}; mkdir -p $OUT
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 $CMD > $OUT/plain_c$CFG.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|rc::' --csv \
    --log-file $OUT/launches_c$CFG.csv $CMD > $OUT/ncu_launches_c$CFG.log 2>&1
echo "launches c$CFG exit $?" >> $OUT/status

#!/bin/bash
# launch list of the default bench command (our kernels), C5 bench line, C4 bench
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
CMD="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 $CMD > $OUT/plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|rc::' --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launches exit $?" >> $OUT/status
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 exit $?" >> $OUT/status
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 exit $?" >> $OUT/status

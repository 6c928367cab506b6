#!/bin/bash
# Trimmed round-end evidence after a change of the curved segment kernel only: smoke, full GPU
# suite, bench lines C4 (default) / C5 / C3, reference arm, ncu launch list of the default bench
# command.  bash tools/gpu_final_short.sh TAG
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/status
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 exit $?" >> $OUT/status
CMD="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 $CMD > $OUT/plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|rc::' --csv \
    --log-file $OUT/launches_c4.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launches exit $?" >> $OUT/status
timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 exit $?" >> $OUT/status
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 exit $?" >> $OUT/status
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "bench ref exit $?" >> $OUT/status

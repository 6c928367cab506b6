#!/bin/bash
# Round-end evidence: smoke, full GPU suite, default bench (C4), C5/C3/C2 bench lines,
# the ncu launch list of the default bench command (our kernels) and a full capture of the
# segment kernel at C4s.
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status
timeout 2400 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/status
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 exit $?" >> $OUT/status
for c in 5 3 2; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; echo "bench c$c exit $?" >> $OUT/status
done
CMD="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 $CMD > $OUT/plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|rc::' --csv \
    --log-file $OUT/launches_c4.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launches exit $?" >> $OUT/status
PCMD="python tools/profile_frame.py --config 45 --frames 2"
timeout 300 $PCMD > $OUT/plain_pf.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cast_curved' -s 1 -c 1 \
    -o $OUT/prof $PCMD > $OUT/ncu_full.log 2>&1
echo "ncu full exit $?" >> $OUT/status

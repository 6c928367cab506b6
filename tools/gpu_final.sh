#!/bin/bash
# Round-end evidence: smoke, full GPU suite, default bench (C4), C5/C3/C2/C1/MB bench lines,
# the ncu launch list of the default bench command (our kernels) and a full capture of the
# segment kernel at C4s.  bash tools/gpu_final.sh TAG
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/status
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 exit $?" >> $OUT/status
timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 exit $?" >> $OUT/status
for c in 3 2 1 6; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; echo "bench c$c exit $?" >> $OUT/status
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "bench ref exit $?" >> $OUT/status
CMD="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 $CMD > $OUT/plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|rc::' --csv \
    --log-file $OUT/launches_c4.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launches exit $?" >> $OUT/status
TCMD="python tools/profile_frame.py --config 4 --frames 1"
timeout 600 $TCMD > $OUT/plain_traffic.log 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:'k_cast_curved|k_prep_slots' --csv --log-file $OUT/traffic_c4.csv $TCMD > $OUT/ncu_traffic.log 2>&1
echo "traffic exit $?" >> $OUT/status
PCMD="python tools/profile_frame.py --config 45 --frames 1"
timeout 300 $PCMD > $OUT/plain_pf.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_cast_curved' -c 1 \
    -o $OUT/prof $PCMD > $OUT/ncu_full.log 2>&1
echo "ncu full exit $?" >> $OUT/status

#!/bin/bash
# One gpurun session: smoke, GPU tests, the default bench, the ncu launch list
# of the bench command (our kernels only) and one `ncu --set full` capture of
# the segment kernel.  Usage (repo root on the GPU box):
#   bash tools/gpu_profile.sh TAG [CONFIG] [STEPS]   (STEPS: all | bench | prof)
set -u
TAG=${1:-run}
CFG=${2:-4}
WHAT=${3:-all}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status
if [ "$WHAT" = all ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/status
fi
if [ "$WHAT" = all ] || [ "$WHAT" = bench ]; then
  timeout 900 python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/status
fi
if [ "$WHAT" = all ] || [ "$WHAT" = prof ]; then
  CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 900 $CMD > $OUT/plain.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|rc::' --csv \
      --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
  echo "launches exit $?" >> $OUT/status
  PCMD="python tools/profile_frame.py --config $CFG --frames 1"
  timeout 600 $PCMD > $OUT/plain_pf.log 2>&1 && \
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_cast_curved|k_cast_affine' \
      -c 1 -o $OUT/prof $PCMD > $OUT/ncu_full.log 2>&1
  echo "ncu full exit $?" >> $OUT/status
fi

#!/bin/bash
# smoke + GPU tests + A/B bench of build variants + ncu full of the segment kernel at C3.
# Usage: [PYTARGET="test files"] bash tools/gpu_round.sh TAG "variants" [pytest-args]
set -u
TAG=$1; VARIANTS=${2:-default}; PYARGS=${3:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status
if [ "$PYARGS" != "skip" ]; then
  timeout 1500 python -m pytest ${PYTARGET:-tests} -m gpu -x -q -rA $PYARGS > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/status
fi
for v in $VARIANTS; do
  if [ "$v" = default ]; then LIB=""; else LIB=$PWD/paper_1809_01334_b200/librc_$v.so; fi
  RC_LIB=$LIB timeout 600 python bench.py --config 4 --steps 5 --no-cpu-baseline > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  echo "bench $v exit $?" >> $OUT/status
done
PCMD="python tools/profile_frame.py --config ${PROFCFG:-45} --frames 1"
timeout 300 $PCMD > $OUT/plain_pf.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cast_curved' -c 1 -o $OUT/prof $PCMD > $OUT/ncu_full.log 2>&1
echo "ncu full exit $?" >> $OUT/status
# DRAM traffic of the segment kernel at the bench's config (one metric pass: no replay of the big buffers)
if [ -n "${TRAFFIC:-}" ]; then
  TCMD="python tools/profile_frame.py --config 4 --frames 3"
  timeout 600 $TCMD > $OUT/plain_traffic.log 2>&1 && \
    timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:'k_cast_curved' -s 2 -c 1 --csv --log-file $OUT/traffic_c4.csv $TCMD > $OUT/ncu_traffic.log 2>&1
  echo "traffic exit $?" >> $OUT/status
fi

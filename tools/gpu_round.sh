#!/bin/bash
# smoke + GPU tests + A/B bench of build variants + ncu full of the segment kernel at C3.
# Usage: bash tools/gpu_round.sh TAG "variants" [pytest-args]
set -u
TAG=$1; VARIANTS=${2:-default}; PYARGS=${3:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status
if [ "$PYARGS" != "skip" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -rA $PYARGS > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/status
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

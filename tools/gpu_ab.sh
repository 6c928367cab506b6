#!/bin/bash
# smoke + pytest subset + C4/C3 (+C5 when C5=1) bench lines without CPU baseline / e2e:
#   bash tools/gpu_ab.sh TAG "PYTEST_K"
set -u
OUT=gpurun_out/$1; K=$2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status
if [ "$K" != "-" ]; then
timeout 1800 python -m pytest tests -m gpu -q -rA -x -k "$K" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/status
fi
timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 exit $?" >> $OUT/status
timeout 900 python bench.py --config 3 --steps 5 --no-cpu-baseline --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "bench c3 exit $?" >> $OUT/status
if [ "${C5:-0}" = 1 ]; then
timeout 1500 python bench.py --config 5 --steps 3 --no-cpu-baseline --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 exit $?" >> $OUT/status
fi

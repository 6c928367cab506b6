#!/bin/bash
# smoke + a pytest subset (+ optional sanitizer tool): bash tools/gpu_quick.sh TAG "PYTEST_K" [TOOL]
set -u
OUT=gpurun_out/$1; K=$2; TOOL=${3:-}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/status
timeout 1800 python -m pytest tests -m gpu -q -rA -x -k "$K" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/status
if [ -n "$TOOL" ]; then bash tools/gpu_sanitize.sh $1 $TOOL; fi

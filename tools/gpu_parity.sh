#!/bin/bash
# GPU parity subset with timings: bash tools/gpu_parity.sh TAG "PYTEST_K"
set -u
OUT=gpurun_out/$1; K=$2; mkdir -p $OUT
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1; free -g > $OUT/free.txt
timeout 3600 python -m pytest tests -m gpu -q -rA -x -k "$K" --durations=0 > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/status

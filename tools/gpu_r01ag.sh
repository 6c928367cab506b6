#!/bin/bash
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_fold_gpu.py tests/test_parity_gpu.py -m gpu -q -x -k "fold or aggregat or c5 or virtual" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/status
for v in default cm8; do
  if [ "$v" = default ]; then LIB=""; else LIB=$PWD/paper_1809_01334_b200/librc_$v.so; fi
  RC_LIB=$LIB timeout 1200 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c5_$v.json 2> $OUT/c5_$v.err; echo "c5 $v exit $?" >> $OUT/status
done
bash tools/gpu_ab2.sh $1 4 - default mb10 mb12

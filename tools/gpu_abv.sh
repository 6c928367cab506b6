#!/bin/bash
# Same-box interleaved A/B of librc build variants on the C4 bench (kernel ms from the JSON line):
#   bash tools/gpu_abv.sh TAG CONFIG ROUNDS variant...   (variant "default" = librc.so, else librc_<variant>.so)
set -u
TAG=$1; CFG=$2; ROUNDS=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in $(seq 1 $ROUNDS); do
  for v in "$@"; do
    if [ "$v" = default ]; then LIB=""; else LIB=$PWD/paper_1809_01334_b200/librc_$v.so; fi
    RC_LIB=$LIB timeout 900 python bench.py --config $CFG --steps 5 --no-cpu-baseline --no-e2e > $OUT/ab_${v}_$r.json 2> $OUT/ab_${v}_$r.err
    echo "$v $r exit $?" >> $OUT/status
  done
done
python - <<PY
import json, glob, collections
res = collections.defaultdict(list)
for f in sorted(glob.glob("$OUT/ab_*.json")):
    v = f.split("/ab_")[1].rsplit("_", 1)[0]
    try:
        d = json.load(open(f)); res[v].append((round(d["roofline"]["kernel_ms"], 1), round(d["ms_per_step"], 1)))
    except Exception as e:
        res[v].append(str(e))
for v, r in res.items(): print(v, r)
PY

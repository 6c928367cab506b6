#!/bin/bash
# The GPU tests against the bounds-checked build (RC_CHECKS device asserts; the
# pool has no compute-sanitizer).  Build first: python -c "from paper_1809_01334_b200
# import build as b; b.build(defines=['RC_CHECKS'], tag='checks')".  bash tools/gpu_checks.sh TAG [PYTEST -k EXPR]
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
K=${2:-}
if [ -n "$K" ]; then KARG=(-k "$K"); else KARG=(); fi
RC_LIB=$PWD/paper_1809_01334_b200/librc_checks.so timeout 3000 python -m pytest tests -m gpu -q "${KARG[@]}" \
  > $OUT/checks_pytest.log 2>&1
echo "checks pytest exit $?" >> $OUT/status

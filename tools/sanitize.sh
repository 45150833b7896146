#!/bin/bash
# compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md), on tools/sanitize_case.py -- the
# small cases that reach every kernel family of the path.  The same command runs natively first.
TOOL=${1:-memcheck}
shift
CASES=${@:-small p20 ahead}
timeout 300 python tools/sanitize_case.py $CASES > gpurun_out/sanitize_native.log 2>&1; rc=$?
echo native_rc=$rc; tail -4 gpurun_out/sanitize_native.log
[ $rc -eq 0 ] || exit 1
EXTRA=""
[ "$TOOL" = "racecheck" ] && EXTRA="--racecheck-report all"
timeout 1500 compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 --error-exitcode 9 \
  python tools/sanitize_case.py $CASES > gpurun_out/sanitize_${TOOL}.log 2>&1
echo "sanitize_${TOOL}_rc=$?"; tail -15 gpurun_out/sanitize_${TOOL}.log
nvidia-smi --query-gpu=index,name,memory.used --format=csv

#!/bin/bash
# One gpurun call: GPU tests, a short bench, then (only if that exited 0) an ncu launch list and
# one `ncu --set full` capture of the hot kernel.  Outputs under gpurun_out/.
# usage: tools/gpu_check.sh [tag] [m for the profiled bench] [kernel regex]
TAG=${1:-chk}; MP=${2:-20000}; KRE=${3:-ozaki_trsm}
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
fi
SMALL="python bench.py --m $MP --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $SMALL > gpurun_out/${TAG}_small.log 2>&1; rc=$?; echo "small_rc=$rc"; tail -1 gpurun_out/${TAG}_small.log | cut -c1-400
if [ $rc -eq 0 ] && [ "${NCU:-1}" = "1" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $SMALL > /dev/null 2>&1; echo "ncu_launch_rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:$KRE -c 1 -o gpurun_out/${TAG}_hot $SMALL > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu_full_rc=$?"
fi

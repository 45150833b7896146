#!/bin/bash
# Full-size (config 2, m=1e6) ncu capture of ONE fused_trsm_gls launch + launch list of a short run.
# The plain command runs first; ncu only if it exited 0 (B200_PROFILING.md rule).
TAG=${1:-r01}
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/${TAG}_plain.log 2>&1; rc=$?; echo "plain_rc=$rc"; tail -1 gpurun_out/${TAG}_plain.log | cut -c1-300
if [ $rc -eq 0 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:fused_trsm -c 1 -o gpurun_out/${TAG}_fused_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu_full_rc=$?"
fi

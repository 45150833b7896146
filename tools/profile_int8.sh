#!/bin/bash
CMD="python bench.py --m 833536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/p2_plain.log 2>&1; rc=$?; echo "plain_rc=$rc"
if [ $rc -eq 0 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p2_launches.csv $CMD > /dev/null 2>&1; echo "ncu_launch_rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:ozaki_trsm -s 16 -c 1 -o gpurun_out/p2_hot $CMD > gpurun_out/p2_ncu.log 2>&1; echo "ncu_full_rc=$?"
fi
timeout 600 python bench.py > gpurun_out/p2_bench.log 2>&1; echo "bench_rc=$?"; tail -1 gpurun_out/p2_bench.log | cut -c1-300
bash tools/run_configs.sh p3

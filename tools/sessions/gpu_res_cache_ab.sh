#!/bin/bash
# Stream/event cache A/B after a full default bench run (the state in which outlier steps appeared):
# 20-step main loops with the host-call log, cache on (default) twice, off (GLS_RES_CACHE=0) twice.
timeout 900 python bench.py > gpurun_out/rc_full.json 2> gpurun_out/rc_full.err; echo full rc=$?
python -c "
import json; d=json.load(open('gpurun_out/rc_full.json')); print(round(d['value']), d['step_ms_rank0'], d['create_ms_rank0'], d['e2e']['value'])"
for mode in on off on off; do
  env=""; [ $mode = off ] && env="GLS_RES_CACHE=0"
  env $env GLS_BENCH_HOSTLOG=1 timeout 900 python bench.py --steps 20 --warmup 3 --no-sub --no-e2e --no-cpu-baseline > gpurun_out/rc_$mode.json 2> gpurun_out/rc_$mode.err; echo rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/rc_$mode.json'))
print('$mode', round(d['ms_per_step'],2), d['step_ms_rank0'])"
  grep "\[host\]" gpurun_out/rc_$mode.err | awk '{if ($3+0 > 40 || $13+0 > 5) print}'
done

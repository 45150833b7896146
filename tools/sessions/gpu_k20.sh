#!/bin/bash
# 20-step main loops (the driver's round-1 K): sampler on vs off, to see steady-state step times and
# whether periodic nvidia-smi queries cost anything.
for mode in on off on off; do
  extra=""; [ $mode = off ] && extra="--no-clocks"
  timeout 900 python bench.py --steps 20 --warmup 3 --no-sub --no-e2e --no-cpu-baseline $extra > gpurun_out/k20_$mode.json 2> gpurun_out/k20_$mode.err; echo rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/k20_$mode.json'))
print('$mode', round(d['value']), round(d['ms_per_step'],2), d['step_ms_rank0'], d['create_ms_rank0'], d['solve_ms_rank0'], d['clocks'])"
done

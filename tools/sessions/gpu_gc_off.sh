#!/bin/bash
# Default bench line three times with cyclic GC off in bench.py (outlier-step check), then one 20-step
# main loop with and one without the clock sampler.
for i in 1 2 3; do
  timeout 900 python bench.py > gpurun_out/gc_$i.json 2> gpurun_out/gc_$i.err; echo rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/gc_$i.json'))
print(round(d['value']), d['step_ms_rank0'], d['create_ms_rank0'], d['solve_ms_rank0'], d['clocks'])"
done
for mode in on off; do
  extra=""; [ $mode = off ] && extra="--no-clocks"
  timeout 900 python bench.py --steps 20 --warmup 3 --no-sub --no-e2e --no-cpu-baseline $extra > gpurun_out/k20_$mode.json 2> gpurun_out/k20_$mode.err; echo rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/k20_$mode.json'))
print('$mode', round(d['value']), round(d['ms_per_step'],2), d['step_ms_rank0'], d['create_ms_rank0'], d['clocks'])"
done

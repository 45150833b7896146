#!/bin/bash
# Default bench line three times with the sampler launched before the warm-up (outlier-step check).
for i in 1 2 3; do
  timeout 900 python bench.py > gpurun_out/se_$i.json 2> gpurun_out/se_$i.err; echo rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/se_$i.json'))
print(d['value'], d['step_ms_rank0'], d['create_ms_rank0'], d['solve_ms_rank0'], d['clocks'])"
done

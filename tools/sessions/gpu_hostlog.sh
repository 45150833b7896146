#!/bin/bash
# Outlier-step diagnosis inside bench.py: host time of every call of the step (GLS_BENCH_HOSTLOG=1).
for i in 1 2; do
GLS_BENCH_HOSTLOG=1 timeout 900 python bench.py --steps 20 --warmup 3 --no-sub --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/hl_$i.json 2> gpurun_out/hl_$i.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/hl_$i.json'))
print(round(d['ms_per_step'],2), d['step_ms_rank0'])"
grep "\[host\]" gpurun_out/hl_$i.err
done

#!/bin/bash
# Outlier-step diagnosis after a full default bench run (pinned host memory of its sub-records freed
# at exit): 20-step main loops with the host-call log and the create's traced phases + pool footprint.
timeout 900 python bench.py > gpurun_out/dt_full.json 2> gpurun_out/dt_full.err; echo full rc=$?
python -c "
import json; d=json.load(open('gpurun_out/dt_full.json')); print(round(d['value']), d['step_ms_rank0'], d['create_ms_rank0'])"
for i in 1 2; do
GLS_TRACE=1 GLS_BENCH_HOSTLOG=1 timeout 900 python bench.py --steps 20 --warmup 3 --no-sub --no-e2e --no-cpu-baseline > gpurun_out/dt_$i.json 2> gpurun_out/dt_$i.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/dt_$i.json'))
print(round(d['ms_per_step'],2), d['step_ms_rank0'])"
grep "\[host\]\|setup alloc\|pool\|chol_inv" gpurun_out/dt_$i.err | paste - - - - | awk '{print}' | head -30
done
free -g; cat /sys/kernel/mm/transparent_hugepage/enabled; nproc

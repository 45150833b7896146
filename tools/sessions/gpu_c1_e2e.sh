#!/bin/bash
# config-1 bench line e2e: GC off (default) twice, GC on once
for v in 0 0 1; do
GLS_BENCH_GC=$v timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c1e_$v.log 2>&1; echo rc=$?
tail -1 gpurun_out/c1e_$v.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']
print('gc=$v', round(d['value']), 'e2e', round(e['value']), 'wall', e['overlap']['wall_ms'], 'fp64host', round(e['fp64_host_input']['value']))"
done
timeout 300 python tools/e2e_steps.py 1 5 2>&1 | tail -6

#!/bin/bash
# Bench lines for configs 1, 3 and 4 (f64 host stream and int8-code stream) into gpurun_out/.
TAG=${1:-cfg}
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/${TAG}_c1.log 2>&1; echo "c1 rc=$?"
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 > gpurun_out/${TAG}_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 python bench.py --config 4 --codes --steps 2 --warmup 1 > gpurun_out/${TAG}_c4codes.log 2>&1; echo "c4codes rc=$?"
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 > gpurun_out/${TAG}_c4.log 2>&1; echo "c4 rc=$?"
for f in c1 c3 c4codes c4; do tail -1 gpurun_out/${TAG}_$f.log | python3 -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['roofline']; e=d.get('e2e') or {}
  print('$f', 'value %.4g' % d['value'], 'ms/step %.1f' % d['ms_per_step'], 'frac %.3f' % r['frac'], 'kernel_ms', r.get('kernel_ms'), 'create', r.get('create_ms'), 'e2e', e.get('value'), 'clk', d['clocks'].get('sm_mhz'))
except Exception as ex: print('$f parse fail', ex)"; done

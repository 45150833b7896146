#!/bin/bash
# Kernel-time sweep of the int8 path over cluster sizes (GLS_OZ_CLUSTER) at config-2 shape.
M=${1:-300000}
for cs in 1 2 4; do
  GLS_OZ_CLUSTER=$cs timeout 300 python bench.py --m $M --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/sweep_cs$cs.log 2>&1
  echo "cs=$cs rc=$? $(tail -1 gpurun_out/sweep_cs$cs.log | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("value %.0f kernel_ms %.2f frac %.3f clocks %s" % (d["value"], r["kernel_ms"], r["frac"], d["clocks"]))' 2>&1)"
done

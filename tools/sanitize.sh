#!/bin/bash
# compute-sanitizer, ONE tool per invocation, on the smoke-size hot path (n=500, m=300).
TOOL=${1:-racecheck}
timeout 600 compute-sanitizer --tool $TOOL --print-limit 20 python __graft_entry__.py smoke > gpurun_out/sanitize_${TOOL}.log 2>&1
echo "sanitize_${TOOL}_rc=$?"; tail -4 gpurun_out/sanitize_${TOOL}.log

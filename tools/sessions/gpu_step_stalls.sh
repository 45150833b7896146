#!/bin/bash
# Outlier-step diagnosis: host timestamps per call, then the same with the create's host phases traced.
timeout 600 python tools/step_stalls.py 25 > gpurun_out/stall_plain.log 2>&1; echo rc=$?
GLS_TRACE=1 timeout 600 python tools/step_stalls.py 25 > gpurun_out/stall_trace.log 2>&1; echo rc=$?
cat gpurun_out/stall_plain.log | grep step
grep -B9 "create  *[4-9][0-9]\.\|create  *[0-9][0-9][0-9]\." gpurun_out/stall_trace.log | head -60

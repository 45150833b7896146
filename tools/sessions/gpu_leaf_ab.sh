#!/bin/bash
# Blocked 128-row leaf (chol_inv_leaf128) vs the round-1 64-row sweeps: parity subset, create A/B, trace.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -k "ragged or config0 or config1_all or not_spd or host_M or dist or repeated or determin" > gpurun_out/leaf_pytest.log 2>&1; echo pytest_rc=$?; tail -4 gpurun_out/leaf_pytest.log
for v in 0 1 0 1; do GLS_LEAF128=$v python tools/bench_create.py 10000 1500 2>&1 | grep create | sed "s/^/leaf128=$v /"; done
GLS_TRACE_CHOL=1 python tools/bench_create.py 10000 2>&1 | tail -13 > gpurun_out/trace_create_leaf128.txt; cat gpurun_out/trace_create_leaf128.txt

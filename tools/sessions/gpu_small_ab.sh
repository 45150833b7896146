#!/bin/bash
# small-product GEMM path (GLS_DGEMM_SMALL) A/B on gls_create, plus the create-related parity subset
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -k "ragged or config0 or config1_all or not_spd or host_M or dist or repeated or determin or gwfgls" > gpurun_out/small_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/small_pytest.log
for v in 0 1 0 1; do GLS_DGEMM_SMALL=$v python tools/bench_create.py 10000 1500 2>&1 | grep create | sed "s/^/small=$v /"; done
GLS_TRACE_CHOL=1 python tools/bench_create.py 10000 1500 2>&1 | grep -E "total|depth|create" > gpurun_out/trace_create_small.txt; cat gpurun_out/trace_create_small.txt

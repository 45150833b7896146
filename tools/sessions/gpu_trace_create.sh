#!/bin/bash
# gls_create main-stream trace (GLS_TRACE_CHOL=1) and standalone create times at n = 1e4 / 1500.
python tools/bench_create.py 10000 1500 2>&1 | grep create
GLS_TRACE_CHOL=1 python tools/bench_create.py 10000 2>&1 | tail -13 > gpurun_out/trace_create_n10000.txt; cat gpurun_out/trace_create_n10000.txt

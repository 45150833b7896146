#!/bin/bash
for v in 0 1; do for n in 128 256 1024; do GLS_LEAF128=$v GLS_TRACE_CHOL=1 python tools/bench_create.py $n 2>&1 | grep -E "total|depth|create" | tail -4 | sed "s/^/leaf128=$v n=$n /"; done; done

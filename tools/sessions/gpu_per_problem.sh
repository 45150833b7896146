#!/bin/bash
# Per-problem int8/FP64 path choice: the path tests, then a config-2 solve timing (no regression check).
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "non_integer or mixed_chunks or per_problem or convert_ahead or large_p or ragged or config0 or host_stream" 2>&1 | tail -4
timeout 600 python tools/ab_solve.py paper_1210_7325_b200/libgls.so 2>&1 | tail -3

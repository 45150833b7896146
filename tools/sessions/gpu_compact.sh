#!/bin/bash
# Compacted FP64 fallback: the path tests, a sparse-dosage timing (1 % of 3e5 SNPs flagged) and the
# config-2 solve timing.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "non_integer or mixed_chunks or per_problem or convert_ahead or large_p or ragged or host_stream or api_async or cached" 2>&1 | tail -3
timeout 600 python tools/sparse_dosage.py 2>&1 | tail -6
timeout 600 python tools/ab_solve.py paper_1210_7325_b200/libgls.so 2>&1 | tail -2

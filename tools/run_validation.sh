#!/bin/bash
# smoke(), the GPU test suite, configs 3 and 4 (int8 codes), and the disk out-of-core runs.
TAG=${1:-val}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 600 python -m pytest tests -m gpu -q -s > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "err|passed|failed" gpurun_out/${TAG}_pytest.log | tail -8
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 > gpurun_out/${TAG}_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 python bench.py --config 4 --codes --steps 2 --warmup 1 > gpurun_out/${TAG}_c4codes.log 2>&1; echo "c4codes rc=$?"
timeout 900 python tools/bench_file_ooc.py --m 1000000 --elem 1 > gpurun_out/${TAG}_file_i8.log 2>&1; echo "file i8 rc=$?"
timeout 900 python tools/bench_file_ooc.py --m 250000 --elem 8 > gpurun_out/${TAG}_file_f64.log 2>&1; echo "file f64 rc=$?"

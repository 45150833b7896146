#!/bin/bash
# GPU session: smoke + the whole GPU test suite + the default bench line (the driver's round-end commands).
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/val_smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/val_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/val_pytest.log
timeout 900 python bench.py > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err; echo bench_rc=$?; tail -c 600 gpurun_out/val_bench.json

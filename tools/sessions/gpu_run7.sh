# GPU session: NEXT-3 tests, multi tests, smoke.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_multi.py -x -q > gpurun_out/r2e_pytest.log 2>&1; echo pytest_rc=$?; tail -30 gpurun_out/r2e_pytest.log

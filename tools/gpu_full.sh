# GPU session: build + smoke + the whole GPU test suite (the driver's round-end commands).
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r2i_pytest.log 2>&1; echo pytest_rc=$?; tail -40 gpurun_out/r2i_pytest.log

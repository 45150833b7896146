# One GPU-box session: host info, build + smoke, the GPU test suite, a short bench (logs under gpurun_out/).
set -x
nproc; free -g; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2a_pytest.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/r2a_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a_bench.log 2>&1; echo bench_rc=$?
tail -c 3000 gpurun_out/r2a_bench.log

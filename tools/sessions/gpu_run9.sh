# GPU session: TMA DGEMM for gls_create -- parity subset, create A/B (GLS_DGEMM_TMA=0/1), ncu DMMA-active.
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -k "ragged or config0 or config1_all or not_spd or host_M or dist or gwfgls or ladder or scaling or repeated" > gpurun_out/r2g_pytest.log 2>&1; echo pytest_rc=$?; tail -25 gpurun_out/r2g_pytest.log
for v in 0 1 0 1; do GLS_DGEMM_TMA=$v python tools/bench_create.py 10000 1500 2>&1 | grep create | sed "s/^/tma=$v /"; done
GLS_TRACE_CHOL=1 python tools/bench_create.py 10000 2>&1 | tail -9
timeout 300 python tools/create_once.py 10000 > gpurun_out/r2g_create_plain.log 2>&1; rc=$?; echo create_rc=$rc
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none --csv --log-file gpurun_out/r2g_create_launches.csv python tools/create_once.py 10000 > gpurun_out/r2g_create_ncu.log 2>&1; echo ncu_create_rc=$?
fi

# GPU session: int8 tensor peak probe, the new stream-report test, create timelines standalone and in-step.
cd tools/umma_probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o peak_i8 peak_i8.cu -lcuda && ./peak_i8 > ../../gpurun_out/r2b_peak_i8.json 2>&1; cd ../..
cat gpurun_out/r2b_peak_i8.json
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stream_report or solve_file or api_async" > gpurun_out/r2b_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/r2b_pytest.log
GLS_TRACE_CHOL=1 GLS_TRACE=1 python tools/bench_create.py 10000 1500 > gpurun_out/r2b_create.log 2>&1; tail -40 gpurun_out/r2b_create.log
GLS_TRACE=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2b_bench_trace.log 2>&1; grep "setup" gpurun_out/r2b_bench_trace.log | tail -8

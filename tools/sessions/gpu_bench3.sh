# GPU session: the bench with its sub-records (N = 1), the 2-process tests, and a functional run of the
# N > 1 bench path (2 ranks on one GPU over gloo; not a measurement).
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -x -q -k "multi or replicate or adopt" > gpurun_out/r2c_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/r2c_pytest.log
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/r2c_bench.log 2>&1; echo bench_rc=$?; tail -c 6000 gpurun_out/r2c_bench.log
GLS_BENCH_DEVICE=0 GLS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --snps 200000 --no-e2e --no-cpu-baseline > gpurun_out/r2c_bench_n2.log 2>&1; echo bench2_rc=$?; tail -c 3000 gpurun_out/r2c_bench_n2.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/r2c_ref_n2.log 2>&1; echo ref2_rc=$?; tail -c 1500 gpurun_out/r2c_ref_n2.log

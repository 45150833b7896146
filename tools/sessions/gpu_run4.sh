# GPU session: gwfgls rung tests + ladder, the N > 1 bench path (2 ranks, gloo, one GPU: functional only),
# the reference arm under torchrun, and the DRAM A/B of the int8 kernel.
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gwfgls or ladder" > gpurun_out/r2d_pytest.log 2>&1; echo pytest_rc=$?; tail -12 gpurun_out/r2d_pytest.log
timeout 900 python tools/ladder.py --n 10000 --m 100000 --m-blackbox 4 --m-gemv 1000 > gpurun_out/r2d_ladder10000.json 2>&1; echo ladder_rc=$?; tail -c 2500 gpurun_out/r2d_ladder10000.json
timeout 900 python tools/ladder.py --n 1500 --m 200000 --m-blackbox 40 --m-gemv 5000 > gpurun_out/r2d_ladder1500.json 2>&1; echo ladder_rc=$?; tail -c 2500 gpurun_out/r2d_ladder1500.json
GLS_BENCH_DEVICE=0 GLS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --snps 200000 --no-e2e --no-cpu-baseline > gpurun_out/r2d_bench_n2.log 2>&1; echo bench2_rc=$?; tail -c 3000 gpurun_out/r2d_bench_n2.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/r2d_ref_n2.log 2>&1; echo ref2_rc=$?; tail -c 1500 gpurun_out/r2d_ref_n2.log
timeout 900 python tools/dram_ab.py > gpurun_out/r2d_dram_ab.json 2>&1; echo dram_rc=$?; cat gpurun_out/r2d_dram_ab.json | tail -c 2000

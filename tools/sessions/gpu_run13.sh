# GPU session: functional N=2 bench path (gloo, one GPU: not a measurement), then the default bench.
python -c "import __graft_entry__ as g; g.build()"
GLS_BENCH_DEVICE=0 GLS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --snps 200000 --no-cpu-baseline > gpurun_out/r2k_bench_n2.log 2>&1; echo bench2_rc=$?; tail -c 1500 gpurun_out/r2k_bench_n2.log
GLS_BENCH_DEVICE=0 GLS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --steps 2 --warmup 1 --snps 200000 --no-cpu-baseline --no-sub --no-e2e --replicate dist > gpurun_out/r2k_bench_n2_dist.log 2>&1; echo bench2dist_rc=$?; tail -c 800 gpurun_out/r2k_bench_n2_dist.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2k_bench.log 2>&1; echo bench_rc=$?; tail -c 300 gpurun_out/r2k_bench.log

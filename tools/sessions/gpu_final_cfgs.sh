#!/bin/bash
# Final-build session: functional N = 2 bench paths (gloo, two ranks on the one GPU: not a measurement),
# then the config 1 / 3 / 4 bench lines.
GLS_BENCH_DEVICE=0 GLS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --snps 200000 --no-cpu-baseline > gpurun_out/fin_bench_n2.log 2>&1; echo bench2_rc=$?; tail -c 600 gpurun_out/fin_bench_n2.log
GLS_BENCH_DEVICE=0 GLS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --steps 2 --warmup 1 --snps 200000 --no-cpu-baseline --no-sub --no-e2e --replicate dist > gpurun_out/fin_bench_n2_dist.log 2>&1; echo bench2dist_rc=$?; tail -c 400 gpurun_out/fin_bench_n2_dist.log
bash tools/run_configs.sh fin

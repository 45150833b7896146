#!/bin/bash
# dist create from the stream-ordered pool: its GPU tests, then the world-1 bench line (--replicate dist)
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --replicate dist --steps 3 --warmup 3 --no-sub --no-e2e --no-cpu-baseline > gpurun_out/dist_w1.json 2> gpurun_out/dist_w1.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/dist_w1.json')); print(round(d['value']), d['step_ms_rank0'], d['create_ms_rank0'])"

#!/bin/bash
# Step-0 box measurements. Output -> gpurun_out/probe.log
set -x
nproc; lscpu | head -20; free -g; numactl -H 2>/dev/null | head -20
nvidia-smi; nvidia-smi topo -m 2>/dev/null | head -20
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/probe/probe
kill $SMI
python -c "
import torch,time
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda');b=torch.randn_like(a)
for _ in range(3): c=a@b
torch.cuda.synchronize();t=time.time()
for _ in range(10): c=a@b
torch.cuda.synchronize();dt=(time.time()-t)/10
print('cuBLAS DGEMM 8192^3: %.2f TFLOP/s'%(2*8192**3/dt/1e12))
"

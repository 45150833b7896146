# A/B of the TMA GEMM tile schedule (cost-ordered snake vs round-robin): bitwise digests + create times
GLS_DGEMM_SCHED=0 python tools/create_digest.py 1500 10000 4097
GLS_DGEMM_SCHED=1 python tools/create_digest.py 1500 10000 4097
for r in 1 2; do
  echo sched=0; GLS_DGEMM_SCHED=0 python tools/bench_create.py 10000 1500
  echo sched=1; GLS_DGEMM_SCHED=1 python tools/bench_create.py 10000 1500
done
GLS_TRACE_GEMM=1 python tools/create_timeline.py 10000 > gpurun_out/tl.log 2> gpurun_out/tl_gemm.log; rm -f gpurun_out/create_trace_n*.json

# A/B: look-ahead (side stream) products after the main stream's L21top / SYRK11 vs concurrently
GLS_SIDE_AFTER=0 python tools/create_digest.py 1500 10000
GLS_SIDE_AFTER=1 python tools/create_digest.py 1500 10000
for r in 1 2; do
  echo after=0; GLS_SIDE_AFTER=0 python tools/bench_create.py 10000 1500
  echo after=1; GLS_SIDE_AFTER=1 python tools/bench_create.py 10000 1500
done
GLS_TRACE_GEMM=1 python tools/create_timeline.py 10000 > gpurun_out/tl.log 2> gpurun_out/tl_gemm.log; rm -f gpurun_out/create_trace_n*.json

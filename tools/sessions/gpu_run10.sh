# GPU session: free-SM budget of the look-ahead GEMMs (GLS_CHOL_FREE_SMS), then the full bench.
python -c "import __graft_entry__ as g; g.build()"
for f in 16 32 48 8 24; do GLS_CHOL_FREE_SMS=$f python tools/bench_create.py 10000 1500 2>&1 | grep create | sed "s/^/free=$f /"; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2h_bench.log 2>&1; echo bench_rc=$?; tail -c 800 gpurun_out/r2h_bench.log

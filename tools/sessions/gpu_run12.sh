# GPU session: the default bench line with every sub-record.
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2j_bench.log 2>&1; echo bench_rc=$?; tail -c 600 gpurun_out/r2j_bench.log

# GPU session: int8 kernel wait profile (GLS_OZ_PROF), bench with the distributed create at N=1,
# ncu of the create's GEMMs and of the int8 kernel (after the plain commands exit 0).
python -c "import __graft_entry__ as g; g.build()"
GLS_OZ_PROF=1 timeout 600 python tools/ab_solve.py paper_1210_7325_b200/libgls.so 1000000 2 > gpurun_out/r2f_ozprof.log 2>&1; echo prof_rc=$?; grep "oz prof" gpurun_out/r2f_ozprof.log | tail -12
timeout 600 python bench.py --steps 3 --warmup 2 --replicate dist --no-e2e --no-cpu-baseline --no-sub > gpurun_out/r2f_bench_dist.log 2>&1; echo bench_dist_rc=$?; tail -c 1500 gpurun_out/r2f_bench_dist.log
timeout 300 python tools/create_once.py 10000 > gpurun_out/r2f_create_plain.log 2>&1; rc=$?; echo create_rc=$rc
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none --csv --log-file gpurun_out/r2f_create_launches.csv python tools/create_once.py 10000 > gpurun_out/r2f_create_ncu.log 2>&1; echo ncu_create_rc=$?
fi
CMD="python bench.py --snps 833536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sub"
timeout 600 $CMD > gpurun_out/r2f_plain.log 2>&1; rc=$?; echo plain_rc=$rc
if [ $rc -eq 0 ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ozaki_trsm -s 16 -c 1 -o gpurun_out/r2f_int8_full $CMD > gpurun_out/r2f_ncu_int8.log 2>&1; echo ncu_int8_rc=$?
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches.csv $CMD > gpurun_out/r2f_ncu_launch.log 2>&1; echo ncu_launch_rc=$?
fi

# A/B: pR > 1 epilogue parks region 0's z block in TMEM so region 1 drains first (GLS_OZ_PARK=1) vs not;
# parity subset first (config-3 shapes), then config 3 timing and the wait profile
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or config3 or p20 or rank_def or repeated" 2>&1 | tail -3
for lib in paper_1210_7325_b200/libgls.so tools/ab_libs/nopark/libgls.so; do
  echo "== $lib"; GLS_OZ_PROF=1 python tools/ab_solve.py $lib 100000 3 2>&1 | grep "oz prof" | tail -1
done
for r in 1 2; do for lib in paper_1210_7325_b200/libgls.so tools/ab_libs/nopark/libgls.so; do
  python tools/ab_solve.py $lib 200000 3 | tail -2; done; done

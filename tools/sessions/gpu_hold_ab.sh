# A/B: stages the int8 MMA issuer may hold for deferred region-1 MMAs (3 = ST-1 default, 2, 1), with the
# in-kernel wait profile (GLS_OZ_PROF) and without it (timing)
for lib in paper_1210_7325_b200/libgls.so tools/ab_libs/hold2/libgls.so tools/ab_libs/hold1/libgls.so; do
  echo "== $lib"; GLS_OZ_PROF=1 python tools/ab_solve.py $lib 300000 2 2>&1 | grep "oz prof" | tail -2
done
for r in 1 2; do for lib in paper_1210_7325_b200/libgls.so tools/ab_libs/hold2/libgls.so tools/ab_libs/hold1/libgls.so; do
  python tools/ab_solve.py $lib 1000000 2 | tail -2; done; done

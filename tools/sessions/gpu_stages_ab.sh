# A/B: a fifth pipeline stage for int8 launches without a convert-ahead job (GLS_OZ_DEEP=1 default) vs
# four stages everywhere (GLS_OZ_DEEP=0); X_R as FP64 (only the block's last chunk changes) and as codes
for r in 1 2; do for dp in 1 0; do
  echo "deep=$dp codes"; GLS_OZ_DEEP=$dp python tools/ab_solve.py paper_1210_7325_b200/libgls.so 1000000 2 i8 | tail -2
  echo "deep=$dp fp64";  GLS_OZ_DEEP=$dp python tools/ab_solve.py paper_1210_7325_b200/libgls.so 1000000 2 | tail -2
done; done
GLS_OZ_PROF=1 python tools/ab_solve.py paper_1210_7325_b200/libgls.so 300000 2 i8 2>&1 | grep "oz prof" | tail -1
GLS_OZ_PROF=1 python tools/ab_solve.py paper_1210_7325_b200/libgls.so 300000 3 i8 2>&1 | grep "oz prof" | tail -1
for dp in 1 0; do echo "deep=$dp config3 codes"; GLS_OZ_DEEP=$dp python tools/ab_solve.py paper_1210_7325_b200/libgls.so 200000 3 i8 | tail -1; done

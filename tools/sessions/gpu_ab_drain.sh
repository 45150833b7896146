# A/B of the int8 epilogue drain (4 vs 2 TMEM round trips per row block), alternating builds on one box.
for r in 1 2; do
  python tools/ab_solve.py paper_1210_7325_b200/libgls.so 1000000 2 2>&1 | tail -3
  python tools/ab_solve.py paper_1210_7325_b200/libgls_rt2.so 1000000 2 2>&1 | tail -3
done
python tools/ab_solve.py paper_1210_7325_b200/libgls.so 500000 3 2>&1 | tail -2
python tools/ab_solve.py paper_1210_7325_b200/libgls_rt2.so 500000 3 2>&1 | tail -2

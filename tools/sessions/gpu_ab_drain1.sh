# A/B of the one-round-trip drain (pR = 1 variants) against the two-round-trip build, one box
for r in 1 2; do
  python tools/ab_solve.py paper_1210_7325_b200/libgls.so
  python tools/ab_solve.py tools/ab_libs/two/libgls.so
done

# A/B: MB of X panels the int8 kernel pins in L2 (GLS_OZ_PIN_MB; default 85)
for r in 1 2; do for mb in 85 40 0 110; do
  echo "pin=$mb"; GLS_OZ_PIN_MB=$mb python tools/ab_solve.py paper_1210_7325_b200/libgls.so 1000000 2 | tail -2
done; done

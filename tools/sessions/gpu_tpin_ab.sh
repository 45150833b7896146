# A/B: digit tiles of the first steps loaded L2::evict_last (GLS_OZ_TPIN_STEPS), with the X pin at 85 or 60 MB
for r in 1 2; do for cfg in "0 85" "30 85" "50 60" "80 50"; do
  set -- $cfg; echo "tpin=$1 xpin=$2"; GLS_OZ_TPIN_STEPS=$1 GLS_OZ_PIN_MB=$2 python tools/ab_solve.py paper_1210_7325_b200/libgls.so 1000000 2 | tail -2
done; done

# A/B: L2 policy of the unpinned X chunk loads: evict_first (default) vs evict_normal (GLS_OZ_XSTREAM=normal)
for r in 1 2 3; do for v in first normal; do
  echo "xstream=$v"; GLS_OZ_XSTREAM=$v python tools/ab_solve.py paper_1210_7325_b200/libgls.so 1000000 2 | tail -2
done; done

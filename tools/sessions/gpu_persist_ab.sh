# A/B: L2 persisting set-aside (cudaLimitPersistingL2CacheSize) with the int8 kernel's evict_last pins
for r in 1 2; do for mb in 0 79 40; do
  echo "persist=$mb"; GLS_L2_PERSIST_MB=$mb python tools/ab_solve.py paper_1210_7325_b200/libgls.so 1000000 2 | tail -2
done; done

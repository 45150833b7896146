# A/B: SMs the off-critical-path products (look-ahead, Y) of gls_create leave to the main stream
for r in 1 2; do
for f in 8 12 16 24 32 48 64; do
  echo free=$f; GLS_CHOL_FREE_SMS=$f python tools/bench_create.py 10000
done
done

# A/B: grid caps (SMs) of the off-critical-path products of gls_create, per stream kind (side = look-ahead,
# aux = Y); default 132 / 132 (16 SMs free each -- but two can run at once)
for r in 1 2; do
for sa in "132 132" "132 66" "66 66" "100 66" "132 100" "100 100" "116 80" "80 116"; do
  set -- $sa; echo "side=$1 aux=$2"; GLS_CAP_SIDE=$1 GLS_CAP_AUX=$2 python tools/bench_create.py 10000
done; done

# A/B: L2 evict_first hints on the convert-ahead traffic (FP64 bulk loads, int8 stores) vs none
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "convert_ahead or config2_full or perturbation" 2>&1 | tail -2
for r in 1 2 3; do for lib in paper_1210_7325_b200/libgls.so tools/ab_libs/nohint/libgls.so; do
  python tools/ab_solve.py $lib 1000000 2 | tail -2; done; done

# A/B: convert-ahead staging buffer size (8 KiB default -> 4 pipeline stages; 1 KiB -> 5 stages fit)
for lib in paper_1210_7325_b200/libgls.so tools/ab_libs/cv1024/libgls.so tools/ab_libs/cv2048/libgls.so; do
  echo "== $lib"; GLS_OZ_PROF=1 python tools/ab_solve.py $lib 300000 2 2>&1 | grep "oz prof" | tail -1
done
for r in 1 2; do for lib in paper_1210_7325_b200/libgls.so tools/ab_libs/cv1024/libgls.so; do
  python tools/ab_solve.py $lib 1000000 2 | tail -2; done; done

#!/bin/bash
# Is the int8 kernel power-bound?  Config-2 solve with the persistent grid capped at 74 (all), 70, 66, 60
# CTA pairs, clocks and power sampled during each run.
for P in 74 66 70 60 74; do
  nvidia-smi -i 0 --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 200 > gpurun_out/pw_$P.smi 2>&1 &
  SMI=$!
  GLS_OZ_PAIRS=$P timeout 600 python tools/ab_solve.py paper_1210_7325_b200/libgls.so 2>&1 | tail -2 | sed "s/^/pairs=$P /"
  kill $SMI
  python3 -c "
import statistics
r=[l.split(',') for l in open('gpurun_out/pw_$P.smi') if l.strip() and l[0].isdigit()]
c=[float(x[0]) for x in r]; p=[float(x[1]) for x in r]
hi=[i for i,x in enumerate(p) if x>700]
print('   pairs=$P clock median under load', statistics.median([c[i] for i in hi]) if hi else None, 'power median', statistics.median([p[i] for i in hi]) if hi else None, 'samples', len(hi))"
done

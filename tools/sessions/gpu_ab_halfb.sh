#!/bin/bash
# L2-throughput test of the int8 kernel: the same solve with half the digit-tile bytes per stage (wrong
# results, timing only) vs the baseline build; plus the resident-cluster counts of the kernel's shape.
./tools/leaf_probe/occ
for lib in base halfb base halfb; do python tools/ab_solve.py tools/ab_libs/libgls_$lib.so 1000000 2 2>&1 | tail -2 | sed "s/^/$lib /"; done

#!/bin/bash
# A/B of int8-kernel variants (tools/ab_libs/libgls_<name>.so) on the config-2 solve, interleaved.
for rep in 1 2; do for lib in "$@"; do python tools/ab_solve.py tools/ab_libs/libgls_$lib.so 1000000 2 2>&1 | tail -2 | sed "s/^/$lib /"; done; done

#!/bin/bash
# r4a: unroll / occupancy variants of the staged coarse-sweep and synthesis kernels (canonical fp64)
out=gpurun_out/r4a_canon_ab.log; : > $out
for cfg in C5 C4; do for lib in u1 u2 u4 mb6 mb5u2 mb8; do
  PDD_LIB=build/ab/c_$lib/libpdd.so timeout 300 python scripts/ab/canon_ab.py --cfg $cfg 2>&1 | grep -E '^\{|rror' >> $out
done; done

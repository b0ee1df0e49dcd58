#!/bin/bash
# r4f: coarse fast path without the in-loop call (v3), synthesis strip kernel with / without its fast path
out=gpurun_out/r4f_canon_v3.log; : > $out
for cfg in C5 C4; do for lib in u1 s8 v3 v3sf v3nf; do
  PDD_LIB=build/ab/c_$lib/libpdd.so timeout 300 python scripts/ab/canon_ab.py --cfg $cfg 2>&1 | grep -E '^\{|rror' >> $out
done; done

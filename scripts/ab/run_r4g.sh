#!/bin/bash
# r4g: coarse sweep with strips of tiles per CTA (table rows staged once per strip), fast path with field-wise reads (v4)
out=gpurun_out/r4g_coarse_strip.log; : > $out
for cfg in C5 C4; do for lib in u1 s8 v4s1 v4s2 v4s3 v4s2nf; do
  PDD_LIB=build/ab/c_$lib/libpdd.so timeout 300 python scripts/ab/canon_ab.py --cfg $cfg 2>&1 | grep -E '^\{|rror' >> $out
done; done

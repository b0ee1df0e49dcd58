#!/bin/bash
# r4d: interior fast path of the synthesis too (build/ab/c_fast2) against the r4a baseline (build/ab/c_u1)
out=gpurun_out/r4d_synth_fast.log; : > $out
for cfg in C5 C4 C2; do for lib in build/ab/c_u1/libpdd.so build/ab/c_fast2/libpdd.so; do
  PDD_LIB=$lib timeout 300 python scripts/ab/canon_ab.py --cfg $cfg 2>&1 | grep -E '^\{|rror' >> $out
done; done

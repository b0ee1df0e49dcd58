#!/bin/bash
# r4e: synthesis as a strip kernel with the table rows staged in shared memory (strip length, interior fast path)
out=gpurun_out/r4e_synth_strip.log; : > $out
for cfg in C5 C4; do for lib in u1 s8 s8f s4 s16f s32f s32; do
  PDD_LIB=build/ab/c_$lib/libpdd.so timeout 300 python scripts/ab/canon_ab.py --cfg $cfg 2>&1 | grep -E '^\{|rror' >> $out
done; done

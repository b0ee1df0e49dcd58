#!/bin/bash
# r4k, r4l: unroll variants on the adopted kernels (strip synthesis, coarse fast path)
out=gpurun_out/r4l_unroll.log; : > $out
for cfg in C5 C4; do for lib in build/ab/c_u1/libpdd.so "" build/ab/c_su8/libpdd.so build/ab/c_cu4/libpdd.so build/ab/c_su8cu3/libpdd.so; do
  PDD_LIB=$lib timeout 300 python scripts/ab/canon_ab.py --cfg $cfg 2>&1 | grep -E '^\{|rror' >> $out
done; done

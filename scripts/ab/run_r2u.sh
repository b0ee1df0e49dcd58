#!/bin/bash
# r2u: 16 x 64 path-3 tiles with 4 warps per CTA (6 CTAs / SM) under the work queue
out=gpurun_out/r2u_th16nw4.log
for cfg in C5 C4 C2; do
  for lib in th16nw4; do for qt in 0 1332 2664 4000; do
    echo "== $cfg $lib qt=$qt" >> $out
    PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy --qt $qt 2>&1 | grep -E '^\{|rror' >> $out
  done; done
  echo "== $cfg th16nw4 static" >> $out
  PDD_LIB=build/ab/th16nw4/libpdd.so timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes static --cols 64 2>&1 | grep -E '^\{|rror' >> $out
done

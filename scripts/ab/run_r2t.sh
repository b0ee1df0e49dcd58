#!/bin/bash
# r2t: 16 x 64 path-3 tiles (dev build -DPDD_P3_TH=16) against 32 x 64 under the work queue
out=gpurun_out/r2t_th16.log
for cfg in C5 C4 C2; do
  for lib in dev th16; do for qt in 0 1332 2664; do
    echo "== $cfg $lib qt=$qt" >> $out
    PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy --qt $qt 2>&1 | grep -E '^\{|rror' >> $out
  done; done
done

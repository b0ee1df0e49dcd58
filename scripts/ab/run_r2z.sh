#!/bin/bash
# r2z: 2 CTAs / SM (up to 128 registers) for the fp32 row-table kernel against 3 CTAs / SM (80 registers)
out=gpurun_out/r2z_mb2.log
for cfg in C5 C4; do for lib in dev mb2; do for qt in 0 888; do
  echo "== $cfg $lib qt=$qt" >> $out
  PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy,static --qt $qt 2>&1 | grep -E '^\{|rror' >> $out
done; done; done

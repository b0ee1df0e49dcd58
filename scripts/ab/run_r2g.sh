#!/bin/bash
# r2g: A/B of the next-tile prefetch (cp.async staging) in the work-queue kernel
out=gpurun_out/r2g_prefetch.log
for cfg in C5 C4 C3 C2; do
  for v in nopref dev; do
    echo "== $cfg $v" >> $out
    PDD_LIB=build/ab/$v/libpdd.so timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy,static 2>&1 | grep -E '^\{|rror|phases' >> $out
  done
done

#!/bin/bash
# r3l: relaxed progress counters (volatile store / load behind compiler barriers, no MEMBAR.CTA)
# against release / acquire in the row pipeline
out=gpurun_out/r3l_relaxed.log
for cfg in C5 C4 C3; do for lib in dev relaxed; do
  echo "== $cfg $lib" >> $out
  PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy,static 2>&1 | grep -E '^\{|rror' >> $out
done; done

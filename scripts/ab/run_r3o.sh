#!/bin/bash
# r3o: next-tile prefetch (cp.async) in the fp32 row-table kernel on the 16 x 64 tiles (C4, C2; dev
# build -DPDD_PREFETCH3=1 turns it on for 32 x 64 and 16 x 64)
out=gpurun_out/r3o_pref_low.log
for cfg in C4 C2 C5; do for lib in dev pref3; do
  echo "== $cfg $lib" >> $out
  PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy,patchy 2>&1 | grep -E '^\{|rror' >> $out
done; done

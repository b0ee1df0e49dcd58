#!/bin/bash
# r3j: nanosleep in the row-pipeline spin-wait (PDD_SPIN_NS) against the plain spin
out=gpurun_out/r3j_spin.log
for cfg in C5 C4; do for lib in dev spin32 spin100; do
  echo "== $cfg $lib" >> $out
  PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy,static 2>&1 | grep -E '^\{|rror' >> $out
done; done

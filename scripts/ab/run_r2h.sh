#!/bin/bash
# r2h: neighbour-activation threshold and active-set size of the work queue (dev build)
export PDD_LIB=build/ab/dev/libpdd.so
out=gpurun_out/r2h_tact.log
for cfg in C5 C4 C3 C2; do
  for ta in 1.0 0.5 0.25; do for w in 2 2.5; do
    echo "== $cfg TACT=$ta QW=$w" >> $out
    PDD_TACT=$ta PDD_QW=$w timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy,static 2>&1 | grep -E '^\{|rror' >> $out
  done; done
done

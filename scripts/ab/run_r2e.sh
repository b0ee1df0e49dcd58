#!/bin/bash
# r2e: work-queue v2 parameter scan (active-set size x sweeps per visit) with the dev build
export PDD_LIB=build/ab/dev/libpdd.so
out=gpurun_out/r2e_scan.log
for cfg in C5 C4 C3 C2; do
  for w in 2 3 4 6 10; do
    echo "== $cfg QW=$w" >> $out
    PDD_QW=$w timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy --k 1,2,1 2>&1 | grep -E '^\{|rror' >> $out
  done
  echo "== $cfg rounds" >> $out
  timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule rounds --modes patchy,static --k 0,0 2>&1 | grep -E '^\{|rror' >> $out
  echo "== $cfg queue static" >> $out
  timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes static --k 0,0,2,8 2>&1 | grep -E '^\{|rror' >> $out
done
for ta in 0.5 0.25; do
  echo "== C5 QW=3 TACT=$ta" >> $out
  PDD_TACT=$ta PDD_QW=3 timeout 300 python scripts/explore.py --cfg C5 --tol 1e-7 --schedule queue --modes patchy --k 1,1 2>&1 | grep -E '^\{|rror' >> $out
done

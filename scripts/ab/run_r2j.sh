#!/bin/bash
export PDD_LIB=build/ab/dev/libpdd.so
out=gpurun_out/r2j_c3.log
for w in 0.75 1.0 1.25 1.5 2.0; do
  echo "== C3 kernel=4 QW=$w" >> $out
  PDD_QW=$w timeout 300 python scripts/explore.py --cfg C3 --tol 1e-7 --schedule queue --kernel 4 --modes patchy,patchy --k 1,2 2>&1 | grep -E '^\{|rror' >> $out
done

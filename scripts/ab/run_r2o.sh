#!/bin/bash
# r2o: queue target rule tiles/25 in [0.75 R, 3 R] and queue tolerance factor (dev build)
export PDD_LIB=build/ab/dev/libpdd.so
out=gpurun_out/r2o_scan.log
for cfg in C5 C4 C3 C2; do
  for v in "" "PDD_QT25=1" "PDD_QTOL=0.8" "PDD_QT25=1 PDD_QTOL=0.8" "PDD_QT25=1 PDD_QTOL=0.9"; do
    echo "== $cfg $v" >> $out
    env $v timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy,patchy,static 2>&1 | grep -E '^\{|rror' >> $out
  done
done

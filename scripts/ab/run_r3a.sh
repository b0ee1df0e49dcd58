#!/bin/bash
# r3a: queue target and sweeps per visit on the final tile geometries (C3: 16 x 64 general tiles,
# C4 / C2: 16 x 64 row-table tiles)
out=gpurun_out/r3a_scan.log
for spec in "C3 300" "C3 444" "C3 592" "C3 888" "C3 1184" "C4 333" "C4 444" "C4 666" "C4 888" "C4 1332" "C2 0" "C2 100"; do
  set -- $spec
  echo "== $1 qt=$2" >> $out
  timeout 300 python scripts/explore.py --cfg $1 --tol 1e-7 --schedule queue --modes patchy --k 1,2,1 --qt $2 2>&1 | grep -E '^\{|rror' >> $out
done

#!/bin/bash
# r2s: path-3 tile geometry under the work queue (patchy): 32x64 (default) against 16x128
out=gpurun_out/r2s_tile.log
for cfg in C5 C4; do
  for c in 64 128; do for qt in 0 1332 2000; do
    echo "== $cfg cols=$c qt=$qt" >> $out
    timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy --cols $c --qt $qt 2>&1 | grep -E '^\{|rror' >> $out
  done; done
done

#!/bin/bash
# r2r: upstream-first service of the work queue (speculative tiles go back, dev build)
export PDD_LIB=build/ab/dev/libpdd.so
out=gpurun_out/r2r_skip.log
for cfg in C5 C4 C2; do
  for v in "PDD_QSKIP=0" "PDD_QSKIP=1" "PDD_QSKIP=2" "PDD_QSKIP=4" "PDD_QSKIP=2 PDD_QSLACK=0.5" "PDD_QSKIP=2 PDD_QSLACK=0.1" "PDD_QSKIP=8 PDD_QSLACK=0.25"; do
    echo "== $cfg $v" >> $out
    env $v timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy 2>&1 | grep -E '^\{|rror' >> $out
  done
done

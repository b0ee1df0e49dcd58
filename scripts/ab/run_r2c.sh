#!/bin/bash
# r2c: work-queue schedule against device-driven rounds on C5 / C4 / C3 (tol 1e-7)
for cfg in C5 C4 C3; do
  for sch in rounds queue; do
    echo "== $cfg $sch" >> gpurun_out/r2c_sched.log
    timeout 600 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule $sch --modes patchy,static >> gpurun_out/r2c_sched.log 2>&1
    timeout 600 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule $sch --modes patchy >> gpurun_out/r2c_sched.log 2>&1
  done
done

#!/bin/bash
# r2d: per-phase cycle breakdown (PDD_TIMING build) of the C5 / C4 patchy and static solves
export PDD_LIB=build/ab/timing/libpdd.so
for cfg in C5 C4; do
  for sch in ${SCHEDS:-rounds queue}; do
    echo "== $cfg $sch" >> gpurun_out/r2d_phases.log
    timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule $sch --modes patchy,patchy,static >> gpurun_out/r2d_phases.log 2>&1
  done
done

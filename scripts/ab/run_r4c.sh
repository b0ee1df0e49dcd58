#!/bin/bash
# r4c: interior fast path of the coarse sweep (product build) against the r4a baseline (build/ab/c_u1): times, SHA of u_c / a*
out=gpurun_out/r4c_canon_fast.log; : > $out
for cfg in C5 C4 C2; do for lib in build/ab/c_u1/libpdd.so ""; do
  PDD_LIB=$lib timeout 300 python scripts/ab/canon_ab.py --cfg $cfg 2>&1 | grep -E '^\{|rror' >> $out
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "coarse or labels or synth or astar" >> $out 2>&1

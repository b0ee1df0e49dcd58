#!/bin/bash
# ncu --set full of the pre-computation kernels at C5: one mid-solve coarse sweep and the synthesis
ncu --set full --import-source on --clock-control none -k regex:k_coarse_sweep_tiles --launch-skip 150 --launch-count 1 \
    -o gpurun_out/prof_r1o_coarse -f python scripts/profile_sweep.py --mode patchy --k 1 --rounds 1 > gpurun_out/r1o_ncu_c.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_synthesize --launch-count 1 \
    -o gpurun_out/prof_r1o_synth -f python scripts/profile_sweep.py --mode patchy --k 1 --rounds 1 > gpurun_out/r1o_ncu_y.log 2>&1
